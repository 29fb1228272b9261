# Full GPU check: tests, smoke, bench line, reference arm, launch list, ncu --set full captures.
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
for k in fwd2_tc colsum_tc select_cluster assign_tc compact_lut compact_entries merge_bucket gather_kernel key_tile_norm; do
ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/full_$k \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_$k.log 2>&1
done
# the weighted merge only has work on a merging input (config M)
python bench.py --config cfgM --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/plain_cfgM.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"merge_bucket|merge_accum|select_kernel|compact_lut" -c 4 -o gpurun_out/full_cfgM \
    python bench.py --config cfgM --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_cfgM.log 2>&1
python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/plain_e2e.log 2>&1 && \
ncu --set full --clock-control none -k regex:"rope_tab_kernel|rope_table64" -c 2 -o gpurun_out/full_rope python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_full_rope.log 2>&1
python tools/bench_decode.py --config cfg3 > gpurun_out/decode_cfg3.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_step --launch-skip 10 -c 1 -o gpurun_out/full_decode_step \
    python tools/bench_decode.py --config cfg3 --steps 20 > gpurun_out/ncu_full_decode.log 2>&1
python tools/bench_diag.py > gpurun_out/diag.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:redundancy_tc -c 1 -o gpurun_out/full_redundancy_tc \
    python tools/bench_diag.py > gpurun_out/ncu_full_diag.log 2>&1
ls gpurun_out
