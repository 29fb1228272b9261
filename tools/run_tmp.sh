python tools/tune_score.py --reps 5
python tools/tune_score.py --reps 40
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu,clocks_event_reasons.active --format=csv
