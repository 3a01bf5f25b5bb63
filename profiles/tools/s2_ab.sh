# A/B of rigid-kernel variants + rigid parity tests (session 2 of round 2)
mkdir -p gpurun_out/s2
python -c "import oracle; oracle.build()" > /dev/null 2>&1
LIBS="libmardyn.so libmardyn_b0.so libmardyn_sv2.so" CFGS="c2 c3" bash profiles/tools/ab.sh > gpurun_out/s2/ab.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "rigid or c2 or c3 or water or golden or guard or mixture" > gpurun_out/s2/pytest_new.log 2>&1
MARDYN_LIB=$PWD/paper_1408_4599_b200/libmardyn_sv2.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "rigid or c3 or golden" > gpurun_out/s2/pytest_sv2.log 2>&1
cat gpurun_out/s2/ab.log; tail -3 gpurun_out/s2/pytest_new.log gpurun_out/s2/pytest_sv2.log
