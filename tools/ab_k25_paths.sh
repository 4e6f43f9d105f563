for mode in param smem generic; do
  case $mode in
    param) env="";;
    smem) env="SMC_DISK_P=2";;
    generic) env="SMC_DISABLE_DISK=1";;
  esac
  for r in 1 2; do
    echo "$mode $(env $env python tools/run_case.py --config c2 --cutoff 25 --particles 20000 --reps 2 2>&1 | tail -1)"
  done
done
