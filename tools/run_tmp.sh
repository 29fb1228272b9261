timeout 300 python -m pytest tests/test_gpu_score_tc.py -q -x 2>&1 | tail -2
python tools/tune_score.py --var EMS_P2_DEBUG=0,2 --var EMS_P2_POLY=0,2,3
