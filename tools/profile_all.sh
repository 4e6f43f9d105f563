#!/bin/bash
# One GPU call's worth of evidence (run from the repo root under gpurun):
# bench lines for every config, the ncu launch list of the C2 bench, and
# --set full captures of K1 (C2, FP64 and FP32) and K2 (C3 at 1e5 walkers/obs).
# Each ncu command runs only after the same command exited 0 without ncu.
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
for c in c2 c1 c3 c4 c5; do
  python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.log 2>&1 || echo "bench $c failed"
done
python bench.py --config c2 --precision fp32 --steps 5 --warmup 3 > gpurun_out/bench_c2_fp32.log 2>&1 || echo "bench c2 fp32 failed"
python bench.py --steps 2 --warmup 3 > gpurun_out/b_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
python tools/run_case.py --config c2 --reps 1 > gpurun_out/rc_c2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ad_particles -c 1 -f -o gpurun_out/k1_c2 \
      python tools/run_case.py --config c2 --reps 1 > gpurun_out/ncu_k1.log 2>&1
python tools/run_case.py --config c3 --particles 100000 --reps 1 > gpurun_out/rc_c3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:bvp_walkers -c 1 -f -o gpurun_out/k2_c3 \
      python tools/run_case.py --config c3 --particles 100000 --reps 1 > gpurun_out/ncu_k2.log 2>&1
python tools/run_case.py --config c2 --precision fp32 --reps 1 > gpurun_out/rc_c2_fp32.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ad_particles -c 1 -f -o gpurun_out/k1_c2_fp32 \
      python tools/run_case.py --config c2 --precision fp32 --reps 1 > gpurun_out/ncu_k1_32.log 2>&1
ls gpurun_out
