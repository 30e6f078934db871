#!/bin/bash
# time the matvec under env-selected kernel variants: scripts/variants.sh "ENV1" "ENV2" ...
for v in "$@"; do
  echo "== $v"
  env $v timeout 300 python bench.py --no-cpu --steps 10 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), d['roofline']['passes_ms'], d['roofline']['whole_matvec']['frac'])"
done
