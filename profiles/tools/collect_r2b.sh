#!/bin/bash
# Round-2 update after the rigid-kernel change (bit compaction, LJ table as kernel parameters):
# bench lines of c2 / c3, their executed FP32 work (M1), ncu --set full of the c2 / c3 force
# kernels, the GPU test suite.  Everything lands in gpurun_out/r2b/.
set -x
O=gpurun_out/r2b; mkdir -p $O
for c in c2 c3; do python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
B="python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
M="gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd2_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul2_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum"
for c in c2 c3; do
  ncu --metrics $M --clock-control none -k regex:k_force --csv --log-file $O/m1_$c.csv $B --config $c > /dev/null 2>&1
  ncu --set full --import-source on --clock-control none -k regex:k_force -s 1 -c 1 -o $O/force_$c -f $B --config $c > /dev/null 2>&1
done
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
tail -2 $O/pytest_gpu.log
