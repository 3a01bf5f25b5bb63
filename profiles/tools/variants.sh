#!/bin/bash
# bench (and check the forces of) the library variants under paper_1408_4599_b200/variants/ (MARDYN_LIB)
for v in base paper_1408_4599_b200/variants/*.so; do
  if [ "$v" = base ]; then lib=""; else lib="MARDYN_LIB=$v"; fi
  env $lib python profiles/tools/dbg_bal.py 2>&1 | head -1 | sed "s|^|$v check: |"
  for c in "$@"; do
    env $lib python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/vb.json 2>gpurun_out/vb.err
    python -c "
import json; d=json.load(open('gpurun_out/vb.json')); r=d['roofline']
print('$v $c', 'MMUPS %.1f'%d['value'], 'force %.4f ms'%r['force_ms'])" 2>/dev/null || echo "$v $c FAILED $(tail -1 gpurun_out/vb.err)"
  done
done
