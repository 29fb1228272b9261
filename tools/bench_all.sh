# Bench lines for the other BASELINE configs (1 GPU), launch lists (time + DRAM bytes) of the
# select / merge / compact kernels at configs 2, 5 and M, and one FULL reference run of config 3
# (no length extrapolation) to validate the reference arm's extrapolation.
for c in cfg1 cfg2 cfg3b cfgM cfg4; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; tail -1 gpurun_out/bench_$c.log | cut -c1-400; done
python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5.log 2>&1; tail -1 gpurun_out/bench_cfg5.log | cut -c1-400
K="select|norms|assign|gather|compact|merge_bucket|merge_accum|key_tile"
for c in cfg2 cfg5 cfgM; do
python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/plain_tail_$c.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"$K" -c 12 --csv \
    --log-file gpurun_out/tail_$c.csv python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_tail_$c.log 2>&1
done
OMP_WAIT_POLICY=passive timeout 1500 python bench.py --impl reference --steps 1 --warmup 0 --sample-len 32768 > gpurun_out/ref_full_cfg3.log 2>&1; tail -1 gpurun_out/ref_full_cfg3.log | cut -c1-900
ls gpurun_out
