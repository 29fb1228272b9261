timeout 300 python -m pytest tests/test_gpu_score_tc.py -q -x 2>&1 | tail -3
python tools/tune_score.py --var EMS_P2_IMPL=1,2
