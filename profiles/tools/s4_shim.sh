# the library's NCCL transport on several processes of one GPU (tests/nccl_shim.c)
mkdir -p gpurun_out/s4
python -c "import oracle; oracle.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_nccl_shim.py -v -x ${SHIM_K:+-k "$SHIM_K"} > gpurun_out/s4/pytest_shim.log 2>&1
tail -60 gpurun_out/s4/pytest_shim.log
