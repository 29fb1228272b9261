# Bench lines for the other BASELINE configs (1 GPU) + a launch list of our kernels.
for c in cfg1 cfg2 cfg3b cfgM cfg4; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; tail -1 gpurun_out/bench_$c.log | cut -c1-400; done
python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5.log 2>&1; tail -1 gpurun_out/bench_cfg5.log | cut -c1-400
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain_l.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"tc_kernel|select|norms|assign|compact|merge_scatter" -c 16 --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_l.log 2>&1
python bench.py --config cfg5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/plain_l5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"select|norms|assign|compact|merge_scatter" -c 8 --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --config cfg5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_l5.log 2>&1
ls gpurun_out
