python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -2
python tools/bench_decode.py --config cfg3
python tools/bench_decode.py --config cfg4 --batch 32
python tools/bench_decode.py --config cfg5 --seq-len 32768
