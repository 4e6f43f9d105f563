#!/bin/bash
# One GPU call's worth of evidence (run from the repo root under gpurun):
# the GPU test suite, bench lines for every config (FP64 and the FP32
# variant), the reference arm's C2 line, the ncu launch list of the C2 bench
# and --set full captures of the hot kernels (K1 C4 at 512 proposals, K1 C5 at
# 2048 particles/obs, K2 C3 at 1e5 walkers/obs).  Every ncu command runs only
# after the same command exited 0 without ncu.  Outputs: gpurun_out/ev_*.
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/ev_pytest_gpu.log 2>&1; tail -1 gpurun_out/ev_pytest_gpu.log
for c in c2 c1 c3 c4 c5; do
  python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/ev_bench_$c.jsonl 2> gpurun_out/ev_bench_$c.err || echo "bench $c failed"
done
for c in c2 c3 c4 c5; do
  python bench.py --config $c --precision fp32 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ev_bench_${c}_fp32.jsonl 2>&1 || echo "bench $c fp32 failed"
done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev_bench_c2_reference.jsonl 2>&1 || echo "reference arm failed"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev_b_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev_launches.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_launch.log 2>&1
python tools/run_case.py --config c4 --particles 512 --reps 1 > gpurun_out/ev_rc_c4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ad_particles -c 1 -f -o gpurun_out/ev_k1_c4 \
      python tools/run_case.py --config c4 --particles 512 --reps 1 > gpurun_out/ev_ncu_k1_c4.log 2>&1
python tools/run_case.py --config c5 --particles 2048 --reps 1 > gpurun_out/ev_rc_c5.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ad_particles -c 1 -f -o gpurun_out/ev_k1_c5 \
      python tools/run_case.py --config c5 --particles 2048 --reps 1 > gpurun_out/ev_ncu_k1_c5.log 2>&1
python tools/run_case.py --config c3 --particles 100000 --reps 1 > gpurun_out/ev_rc_c3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:bvp_walkers -c 1 -f -o gpurun_out/ev_k2_c3 \
      python tools/run_case.py --config c3 --particles 100000 --reps 1 > gpurun_out/ev_ncu_k2_c3.log 2>&1
ls gpurun_out | grep ev_
