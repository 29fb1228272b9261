for i in 1 2 3; do python bench.py --config cfg5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-200; done
compute-sanitizer --tool memcheck python bench.py --config cfg5 --seq-len 8192 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/memcheck.log 2>&1; grep -E "ERROR SUMMARY|Invalid|at 0x|by thread" gpurun_out/memcheck.log | head -20
