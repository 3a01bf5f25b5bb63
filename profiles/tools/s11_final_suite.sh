# the final binary: smoke() and the whole GPU suite
mkdir -p gpurun_out/s11
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s11/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s11/pytest_gpu.log 2>&1
tail -1 gpurun_out/s11/smoke.log; tail -3 gpurun_out/s11/pytest_gpu.log
