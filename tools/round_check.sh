# Full GPU check: tests, bench line, reference arm, launch list, ncu --set full captures.
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
for k in fwd_tc colsum_tc select_kernel assign_tc compact_lut compact_entries merge_scatter gather_kernel; do
ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/full_$k \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_$k.log 2>&1
done
python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/plain_e2e.log 2>&1 && \
ncu --set full --clock-control none -k regex:rope_kernel -c 1 -o gpurun_out/full_rope python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_full_rope.log 2>&1
ls gpurun_out
