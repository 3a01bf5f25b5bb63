#!/bin/bash
# Final state of round 2 (session 2): smoke, the bench lines of all five configurations and the
# reference arm, and for the changed rigid kernel (c2): executed FP32 work (M1), ncu --set full,
# the launch list.  Everything lands in gpurun_out/s2final/.
set -x
O=gpurun_out/s2final; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
python bench.py > $O/bench_c1.json 2> $O/bench_c1.err
for c in c0 c2 c3 c4; do python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
B="python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
M="gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd2_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul2_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum"
ncu --metrics $M --clock-control none -k regex:k_force --csv --log-file $O/m1_c2.csv $B --config c2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c2_launches.csv $B --config c2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_force -s 1 -c 1 -o $O/force_c2 -f $B --config c2 > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_force -s 1 -c 1 --csv --log-file $O/traffic_c2.csv $B --config c2 > /dev/null 2>&1
tail -1 $O/smoke.log
for c in c0 c1 c2 c3 c4; do python -c "
import json; d=json.load(open('$O/bench_$c.json')); r=d['roofline']
print('$c', round(d['value'],1), 'MMUPS', round(d['ms_per_step']*1e3,1), 'us/step force', round(r['force_ms']*1e3,1), 'frac', round(r['frac'],4), 'e2e', round(d['e2e']['value'],1), 'clk', d['clocks']['sm_mhz'], d['clocks'].get('reasons'))"; done
python -c "import json; d=json.load(open('$O/bench_reference.json')); print('reference', d['value'], d['cpu_baseline'])"
python profiles/tools/m1.py $O/m1_c2.csv
