#!/bin/bash
# A/B bench: each line of $AB_ARGS (';'-separated) is one bench.py argument set.
mkdir -p gpurun_out
: > gpurun_out/ab.log
IFS=';' read -ra SETS <<< "${AB_ARGS:-}"
for a in "${SETS[@]}"; do
  echo "== $a" >> gpurun_out/ab.log
  timeout 600 python bench.py $a 2>&1 | grep -E '^\{|Error|error' | python -c "
import sys, json
for l in sys.stdin:
    try:
        j = json.loads(l); print(j.get('value'), j.get('ms_per_step'), j.get('e2e', {}).get('value'), j.get('dense', {}) if 'dense' in j else '', j.get('speedup_vs_dense', ''))
    except Exception: print(l.strip()[:300])
" >> gpurun_out/ab.log
done
cat gpurun_out/ab.log
