#!/bin/bash
# Round-2 evidence on one B200: bench lines, ncu launch lists and --set full captures of the force
# kernels, executed FP32 work (M1), bandwidth kernels, decomposed-run per-rank timings, full-length
# trajectory parity.  Everything lands in gpurun_out/r2/.
set -x
O=gpurun_out/r2; mkdir -p $O
python bench.py > $O/bench_c1.json 2> $O/bench_c1.err
for c in c0 c2 c3 c4; do python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
B="python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c1_launches.csv $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c2_launches.csv $B --config c2 > /dev/null 2>&1
M="gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd2_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul2_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum"
for c in c1 c2 c3; do
  ncu --metrics $M --clock-control none -k regex:k_force --csv --log-file $O/m1_$c.csv $B --config $c > /dev/null 2>&1
done
for c in c1 c2 c3; do
  ncu --set full --import-source on --clock-control none -k regex:k_force -s 1 -c 1 -o $O/force_$c -f $B --config $c > /dev/null 2>&1
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv -k regex:"k_canon|k_scatter|k_scan|k_integrate|k_finalize" --log-file $O/bw_c1.csv $B > /dev/null 2>&1
python profiles/tools/dd_ranks.py scale c4 1 2 4 8 > $O/dd_c4.log 2>&1
python profiles/tools/dd_ranks.py static c4 8 > $O/dd_static.log 2>&1
python profiles/tools/dd_ranks.py scale c1 2 4 8 > $O/dd_c1.log 2>&1
DD_STEPS=2 DD_WARM=2 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/dd_c4_p8_launches.csv python profiles/tools/dd_ranks.py one c4 8 > /dev/null 2>&1
python profiles/tools/longrun.py c0:10 c1s:100 c2s:100 c3s:100 c4s:200 c1:100 > $O/longrun.log 2>&1
MARDYN_LIB=paper_1408_4599_b200/libmardyn_stats.so python profiles/tools/lj1_stats.py c1 c4 > $O/lj1_stats.log 2>&1
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
tail -2 $O/pytest_gpu.log
