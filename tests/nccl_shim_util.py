"""Build helper for tests/nccl_shim.c (test infrastructure: an NCCL-API stand-in that lets
several processes of a decomposed run share one GPU; see the file's header)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "nccl_shim.c")


def build_shim(outdir):
    """Compile the shim into outdir/libnccl_shim.so (gcc; nccl.h and cuda_runtime.h for the
    types only: the shim links neither NCCL nor CUDA, it dlopens libcuda.so.1)."""
    out = os.path.join(str(outdir), "libnccl_shim.so")
    cuda_inc = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "include")
    subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-std=gnu11", "-I", cuda_inc, "-o", out, SRC, "-ldl"])
    return out
