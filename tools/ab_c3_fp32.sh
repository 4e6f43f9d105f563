for lib in paper_1808_10580_b200/lib/ab/bvp_noahead.so tree; do
  if [ "$lib" = tree ]; then unset SMC_LIBRARY; else export SMC_LIBRARY=$PWD/$lib; fi
  echo "$lib fp32 $(python bench.py --config c3 --precision fp32 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d["ms_per_step"],2))')"
done
unset SMC_LIBRARY
