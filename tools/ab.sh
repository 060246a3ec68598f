#!/bin/bash
# Interleaved A/B of library variants on one box:
#   tools/ab.sh OUT ROUNDS SHAPES VARIANT_A VARIANT_B [...]
# A variant is "-" (the in-tree libmoe.so with the default switches) or a space-separated list
# of VAR=value settings (e.g. "MOE_LIB_PATH=scratch/libX.so MOE_PREFETCH_NEXT=0"). One
# bench_shapes.py JSON line per (round, variant, shape), tagged with the variant, appended to OUT.
out=$1; rounds=$2; shapes=$3; shift 3
for r in $(seq 1 "$rounds"); do
  for v in "$@"; do
    if [ "$v" = "-" ]; then envs=""; else envs="$v"; fi
    env $envs timeout 600 python bench_shapes.py --shapes "$shapes" --steps 2000 2>/dev/null |
      python -c "import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        j=json.loads(l); j['variant']='$v'; j['round']=$r; print(json.dumps(j))" >> "$out"
  done
done
