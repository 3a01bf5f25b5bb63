# system-scope fences after IPC puts: the NCCL stand-in tests and the loopback decomposition tests
mkdir -p gpurun_out/s12
python -c "import oracle; oracle.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_nccl_shim.py tests/test_gpu_decomp.py -q > gpurun_out/s12/pytest.log 2>&1
tail -3 gpurun_out/s12/pytest.log
