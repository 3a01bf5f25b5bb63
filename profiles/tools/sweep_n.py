"""O(N) sweep (Fig. 4) and the 1-GPU decomposition-path
overhead on one B200.

X2: homogeneous single-site LJTS at the paper's state point (T = 0.95, rho = 0.6223, rc = 2.5)
on jittered FCC lattices from 4 000 to 16.7 M molecules; time per molecule-update of the whole
step (`mardyn_step(1)`, one CUDA graph), CUDA events on the context stream, back-to-back steps
(no L2 flush: the small systems live in L2, as the paper's small systems live in cache).
X4: with one rank the decomposition is the plain path by construction (the library takes the
decomposed step only for p >= 2), so the analogue of the paper's sequential-vs-MPI overhead
is the decomposed step with p = 2 loopback ranks on the one GPU (halo molecules, exchange
packing in the force kernel, segment copies, import, two rebuilds; the two ranks run one after
another) against the plain path, at 1 M molecules.

Usage: python profiles/tools/sweep_n.py > profiles/r1_sweep_n.md
"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402
import scenarios as S  # noqa: E402
from paper_1408_4599_b200 import mardyn  # noqa: E402


def time_steps(step, stream, k):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        a.record(stream)
        for _ in range(k):
            step(1)
        b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


def main():
    print("# O(N) sweep and decomposition-path overhead (one B200)\n")
    print(__doc__.split("Usage")[0].strip().replace("\n", " ") + "\n")
    print("| molecules | us / step | ns / molecule-update | MMUPS |")
    print("|---|---|---|---|")
    for nc in (10, 16, 25, 40, 64, 101, 128, 161):
        s = S.lj_fcc(nc, 0.6223, 0.95, 11, f"sweep{nc}", 10)
        n = len(s["r"])
        stream = torch.cuda.Stream()
        ctx = mardyn.from_system(s, stream=stream)
        for _ in range(5):
            ctx.step(1)
        k = 200 if n < 300_000 else 40
        ms = time_steps(ctx.step, stream, k)
        print(f"| {n:,} | {ms * 1e3:.1f} | {ms * 1e6 / n:.3f} | {n / ms / 1e3:.0f} |", flush=True)
        del ctx
        torch.cuda.empty_cache()

    print("\n## X4: plain path vs decomposition path, p = 2 on one GPU (1 048 576 molecules)\n")
    s = S.lj_fcc(64, 0.6223, 0.95, 11, "x4", 10)
    n = len(s["r"])
    stream = torch.cuda.Stream()
    ctx = mardyn.from_system(s, stream=stream)
    for _ in range(5):
        ctx.step(1)
    plain = time_steps(ctx.step, stream, 40)
    del ctx
    with torch.cuda.stream(stream):
        run = mardyn.DecomposedRun(s, 2, transport="loopback", stream=stream)
    for _ in range(5):
        run.step(1)
    dd = time_steps(run.step, stream, 40)
    print("| path | us / step | overhead |")
    print("|---|---|---|")
    print(f"| plain (`mardyn_step`, one graph) | {plain * 1e3:.1f} | |")
    print(f"| decomposed, p = 2 loopback ranks (async step, both ranks' work) | {dd * 1e3:.1f} | "
          f"{(dd / plain - 1) * 100:+.1f} % |")


if __name__ == "__main__":
    main()
