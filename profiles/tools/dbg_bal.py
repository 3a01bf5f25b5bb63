import sys, numpy as np
sys.path.insert(0,'.')
import oracle, scenarios as S
from paper_1408_4599_b200 import mardyn as md
s=S.config1(28)
ctx=md.from_system(s)
F,_=ctx.get_forces()
o=oracle.System(s)
Fo,_,tot=o.forces(s["comp"],o.quantize(s["r"]),s["q"],mode="full")
err=np.abs(F-Fo).max(axis=1); rms=np.sqrt(np.mean(np.sum(Fo**2,1)))
print("N",len(F),"max err/rms",err.max()/rms, "bad",(err>1e-4*rms).sum(), "nan", np.isnan(F).sum())
bad=np.nonzero(err>1e-4*rms)[0][:10]
print(bad, F[bad[:3]] if len(bad) else None, Fo[bad[:3]] if len(bad) else None)
ctx.compute_forces(); ob=ctx.get_observables(); print(ob["n_pairs"], tot["npairs"], ob["U_pot"], tot["U"])
