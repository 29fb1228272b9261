python -m pytest tests/test_gpu_host_pipeline.py tests/test_gpu_rope.py tests/test_gpu_parity.py tests/test_gpu_score_tc.py -x -q 2>&1 | tail -15
for c in 1 2 4 8; do python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-chunks $c 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($c, d['ms_per_step'], d['e2e'])"; done
