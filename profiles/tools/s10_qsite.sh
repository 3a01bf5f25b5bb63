# water: partner charges from the kernel parameters instead of the staged slots (A/B) + c3 parity
mkdir -p gpurun_out/s10
python -c "import oracle; oracle.build()" > /dev/null 2>&1
LIBS="libmardyn.so libmardyn_b0.so" CFGS="c3" bash profiles/tools/ab.sh > gpurun_out/s10/ab.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -k "c3 or rigid or golden or tiny or guard or water or decomp" > gpurun_out/s10/pytest.log 2>&1
cat gpurun_out/s10/ab.log; tail -2 gpurun_out/s10/pytest.log
