# Device ms per config-2 step for environment-knob variants (diagnostics):
#   bash tools/knob_sweep.sh "X=1" "MPO_B200_JFLOOR=16" ...
for v in "$@"; do
  echo "== $v"
  env $v python bench.py --no-batched --no-conversion --no-c3 --no-cpu-baseline --steps 3 --warmup 2 2>/dev/null \
    | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],1))"
done
