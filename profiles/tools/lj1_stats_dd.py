"""LJ1 main-loop statistics of the ranks of a decomposed run (profiling build, see lj1_stats.py)."""
import sys
sys.path.insert(0, ".")
import scenarios as S
from paper_1408_4599_b200 import mardyn
s = S.config(sys.argv[1])
run = mardyn.DecomposedRun(s, int(sys.argv[2]), transport="loopback")
run.step(3)
run.observables()
for c in run.ctxs:
    c.close()
