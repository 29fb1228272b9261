timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"select|compact_lut" -c 4 --csv --log-file gpurun_out/ls.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
grep -E "duration" gpurun_out/ls.csv | awk -F'","' '{print $5, $NF}' | cut -c1-40,150-
