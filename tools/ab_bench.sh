#!/bin/bash
# A/B of library builds on one box: tools/ab_bench.sh CONFIG ROUNDS LIB...
# Runs bench.py --config CONFIG once per library per round (interleaved, so
# clock/thermal drift hits every build alike) and prints ms_per_step per run.
# A LIB of "tree" means the in-tree build.
cfg=$1; rounds=$2; shift 2
for r in $(seq 1 "$rounds"); do
  for lib in "$@"; do
    if [ "$lib" = tree ]; then unset SMC_LIBRARY; else export SMC_LIBRARY=$PWD/$lib; fi
    ms=$(python bench.py --config "$cfg" --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d["ms_per_step"],2), d["clocks"]["sm_mhz"])')
    echo "round $r $lib $ms"
  done
done
unset SMC_LIBRARY
