# full GPU suite + quick bench of the rigid configs with the site-virial build
mkdir -p gpurun_out/s3
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s3/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s3/pytest_gpu.log 2>&1
LIBS="libmardyn.so libmardyn_b0.so" CFGS="c2 c3" bash profiles/tools/ab.sh > gpurun_out/s3/ab.log 2>&1
tail -1 gpurun_out/s3/smoke.log; tail -3 gpurun_out/s3/pytest_gpu.log; cat gpurun_out/s3/ab.log
