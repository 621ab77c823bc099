import sys, numpy as np
sys.path.insert(0, '.')
from paper_2403_03605_b200 import capi, configs as cf
from paper_2403_03605_b200.pd import PDSolver, Scenario
sc = Scenario(cf.get("cfg3"))
s = PDSolver.from_scenario(sc, mode=capi.FAST, device=0).find_pe_pairs()
def run(tag):
    s.initial_acceleration(sc.load_scale(0.0))
    s.step(sc.scales(1, 5))
    t=[]; k=6
    for r in range(8):
        t.append(s.step_timed(sc.scales(k, 20))/20*1e3); k+=20
    print(tag, ["%.2f"%x for x in t], flush=True)
run("fresh handle ")
z = np.zeros(s.n_dof)
s.set_state(z, z, z)
run("same handle, state reset to rest")
s.set_state(z, z, z)
run("again")
