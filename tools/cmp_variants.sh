#!/bin/bash
# Compare library variants on the c2 bench (device ms/step, Jacobi kernel ms) and batched c5.
# usage: tools/cmp_variants.sh base name1 name2 ...   (base = the regular build)
cd "$(dirname "$0")/.."
for v in "$@"; do
  if [ "$v" = base ]; then unset MPO_B200_LIB; else export MPO_B200_LIB=paper_1707_07803_b200/lib/variants/libmpo_b200_$v.so; fi
  echo "== $v"
  python bench.py --no-cpu-baseline --no-conversion $BENCH_EXTRA 2>&1 | grep -E "bench\]|^\{" | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); b=d.get('tnrsvd_batched',{})
        print(round(d['ms_per_step'],1), 'e2e', round(d['e2e']['value'],3), {k: round(x,1) for k,x in d['roofline']['jacobi_ms_per_step'].items()}, 'batched', round(b.get('value',0),2))
    else: print(l.strip())"
done
