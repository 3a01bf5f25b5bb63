#!/bin/bash
# quick bench lines of the given configs (force time and MMUPS), for kernel iteration
for c in "$@"; do
  python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err
  python -c "
import json,sys
d=json.load(open('gpurun_out/b_$c.json')); r=d['roofline']
print('$c', 'MMUPS %.1f'%d['value'], 'step %.4f ms'%d['ms_per_step'], 'force %.4f ms'%r['force_ms'], 'frac %.4f'%r['frac'], 'clk', d['clocks']['sm_mhz'])" || tail -5 gpurun_out/b_$c.err
done
