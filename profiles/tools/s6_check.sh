# full GPU suite after the IPC puts, then the full-size N > 1 bench path through the stand-in
mkdir -p gpurun_out/s6
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s6/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s6/pytest_gpu.log 2>&1
tail -1 gpurun_out/s6/smoke.log; tail -3 gpurun_out/s6/pytest_gpu.log
bash profiles/tools/s5_bench_shim.sh
