"""B200-native ls1-mardyn hot path (arXiv:1408.4599): linked-cell
rigid-molecule force/torque computation, per-step counting-sort cell
rebuild, leapfrog + quaternion rotational integrator, as hand-written
sm_100a CUDA behind the C ABI of include/mardyn.h.

``paper_1408_4599_b200.mardyn`` is the ctypes binding; the library is built
in-tree by ``paper_1408_4599_b200.build``.  This package never imports the
CPU oracle (oracle/), which is test infrastructure only.
"""
__all__ = ["mardyn", "build"]
