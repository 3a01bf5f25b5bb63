# SYM instance staging only the axis slot: A/B against the previous SYM build, rigid parity
mkdir -p gpurun_out/s9
python -c "import oracle; oracle.build()" > /dev/null 2>&1
LIBS="libmardyn.so libmardyn_b0.so" CFGS="c2" bash profiles/tools/ab.sh > gpurun_out/s9/ab.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -k "c2 or rigid or golden or 2clj or tiny or guard or longrun" > gpurun_out/s9/pytest.log 2>&1
cat gpurun_out/s9/ab.log; tail -2 gpurun_out/s9/pytest.log
