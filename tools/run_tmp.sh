python tools/tune_score.py --reps 10 --var EMS_LIB_PATH=_variants/dbg2.so --var EMS_P2_DEBUG=0,2,5,6 --var EMS_P2_POLY=0,2
