"""Main-loop lane balance of the single-site kernel (build with -DMD_LJ1_STATS as
libmardyn_stats.so; MARDYN_LIB points the binding at it): useful candidate pairs over
executed pair slots (32 x the longest lane's list per sub-chunk)."""
import sys
sys.path.insert(0, ".")
import scenarios as S
from paper_1408_4599_b200 import mardyn
for name in sys.argv[1:]:
    s = S.config(name)
    ctx = mardyn.from_system(s)
    ctx.step(2)
    ctx.get_observables()
    print(name, flush=True)
    ctx.close()
