# A/B by environment: ab_env.sh CONFIG ROUNDS "ENV1" "ENV2" ...  ("-" = none)
cfg=$1; rounds=$2; shift 2
for r in $(seq 1 "$rounds"); do
  for e in "$@"; do
    envs=""; [ "$e" != "-" ] && envs="$e"
    ms=$(env $envs python bench.py --config "$cfg" --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d["ms_per_step"],2), d["clocks"]["sm_mhz"])')
    echo "round $r [$e] $cfg $ms"
  done
done
