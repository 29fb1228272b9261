# usage: bash tools/ncu_score.sh <kernel-regex> <out-name> [extra bench args]
# one full ncu capture (source-level, -lineinfo build) of the first launch matching the regex in a
# one-step config-3 bench run; the plain run must exit 0 first (recipe, B200_PROFILING.md)
K=${1:-fwd2_tc}; OUT=${2:-prof}; shift 2
python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e "$@" > gpurun_out/plain_$OUT.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/$OUT \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e "$@" > gpurun_out/ncu_$OUT.log 2>&1
tail -2 gpurun_out/ncu_$OUT.log
