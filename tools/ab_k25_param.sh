for r in 1 2; do
 echo "smem  $(python tools/run_case.py --config c2 --cutoff 25 --particles 20000 --reps 2 2>&1 | tail -1)"
 echo "param $(SMC_DISK_PARAM=1 python tools/run_case.py --config c2 --cutoff 25 --particles 20000 --reps 2 2>&1 | tail -1)"
done
