for c in cfg2 cfg5; do
python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain_$c.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"tc_kernel|select|norms|assign|compact|merge_scatter" -s 8 -c 8 --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$c.log 2>&1
done
