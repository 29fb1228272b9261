# usage: bash tools/ncu_score.sh <kernel-regex> <out-name> [ENV=VAL ...]
K=${1:-fwd_tc}; OUT=${2:-prof}; shift 2; for kv in "$@"; do export "$kv"; done
python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/plain_$OUT.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/$OUT \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$OUT.log 2>&1
tail -2 gpurun_out/ncu_$OUT.log
