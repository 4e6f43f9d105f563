#!/bin/bash
# compute-sanitizer over small cases of every kernel family (run from the repo
# root under gpurun, one tool per call):  tools/sanitize.sh memcheck|racecheck|synccheck
# Each case first runs once without the sanitizer (it must exit 0), then
# under it; the summary line of each run goes to gpurun_out/sanitize_<tool>.log.
tool=${1:-memcheck}
out=gpurun_out/sanitize_$tool.log
mkdir -p gpurun_out; : > "$out"
cases=(
  "--config c2 --particles 2048"                          # K1 disk kernel, parameter-bank coefficients
  "--config c2 --particles 1024 --lattice"                # K1 generic tiled kernel (shared-memory table)
  "--config c2 --particles 1024 --precision fp32"         # K1 FP32 packed FFMA2
  "--config c2 --particles 256 --precision fp64_strict"   # K1 strict (reference order)
  "--config c1"                                           # K1 small launch, shipped config
  "--config c3 --particles 2000"                          # K2 walkers + compaction + K3 tree
  "--config c3 --particles 500 --precision fp32"          # K2 FP32
  "--config c3b --particles 500"                          # K2 with the disk velocity series
  "--config c4 --particles 6"                             # batched K1 (6 proposals) + device pack
  "--config c5 --particles 64"                            # K1 tiled, K=80 (M=10040)
  "--config pcn --particles 4"                            # device-resident pCN chains (CUDA graphs)
  "--config galerkin --cutoff 6"                          # Galerkin reference solver
)
export PCN_STEPS=20
for c in "${cases[@]}"; do
  if ! timeout 300 python tools/run_case.py $c --reps 1 > /dev/null 2>&1; then
    echo "[$c] plain run failed; skipped" | tee -a "$out"; continue
  fi
  timeout 1200 compute-sanitizer --tool "$tool" --print-limit 10 --error-exitcode 9 \
      python tools/run_case.py $c --reps 1 > gpurun_out/san_tmp.log 2>&1
  rc=$?
  summary=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|error" gpurun_out/san_tmp.log | tail -3 | tr '\n' ' ')
  echo "[$c] rc=$rc $summary" | tee -a "$out"
  [ $rc -ne 0 ] && cp gpurun_out/san_tmp.log "gpurun_out/san_fail_${tool}_$(echo $c | tr ' -' '__').log"
done
rm -f gpurun_out/san_tmp.log
