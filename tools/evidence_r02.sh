#!/bin/bash
# Round-2 evidence refresh (run from the repo root under gpurun): GPU suite,
# bench lines C1-C5 (FP64 + FP32), reference arm C2 and C3, ncu launch lists
# of the C2 and C3 benches.  Outputs gpurun_out/ev_*.
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
python bench.py --config c3 --impl reference --steps 3 --warmup 3 > gpurun_out/ev_bench_c3_reference.jsonl 2>&1 || echo "reference arm c3 failed"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev_b_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev_launches.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_launch.log 2>&1
python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev_b3_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev_launches_c3.csv \
      python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_launch_c3.log 2>&1
ls gpurun_out | grep ev_ | wc -l
