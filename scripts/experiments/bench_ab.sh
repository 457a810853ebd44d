# Sustained bench A/B of env knob settings, interleaved: bash bench_ab.sh REPS "workload:steps ..." "SET1" "SET2" ...
reps=$1; works=$2; shift 2
for r in $(seq $reps); do for w in $works; do IFS=: read W S <<< "$w"; for s in "$@"; do
  out=$(env $s python bench.py --workload $W --steps $S --warmup 20 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  echo "$W [$s] $(echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], 'TF', d['ms_per_step'], 'ms', d['clocks']['sm_mhz'], 'MHz', d['clocks'].get('power_w_max'), 'W')")"
done; done; done
