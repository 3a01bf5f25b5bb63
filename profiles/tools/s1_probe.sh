set -x
mkdir -p gpurun_out/s1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s1/build.log 2>&1
bash profiles/tools/bench_quick.sh c1 c2 c3 > gpurun_out/s1/quick.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_force_rigid3 -s 3 -c 1 -o gpurun_out/s1/rig_c2 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/s1/ncu_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_force_lj1 -s 3 -c 1 -o gpurun_out/s1/lj1_c1 python bench.py --config c1 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/s1/ncu_c1.log 2>&1
cat gpurun_out/s1/quick.log
