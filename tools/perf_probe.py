"""Quick timing of device cycles with a per-kernel-class breakdown."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_14208_b200 import configs as CF, _lib
from paper_2207_14208_b200.transfer import build_hierarchy
from paper_2207_14208_b200.solver import MultigridSolver

def probe(setup, cycles=5):
    t0 = time.time()
    levels = build_hierarchy(setup.grid, setup.phi, setup.faces, coarsest_min=setup.coarsest_min)
    t1 = time.time()
    s = MultigridSolver(levels, setup.spec, setup.smoother, setup.cycle, setup.default_variant)
    if setup.f_seed is not None:
        s.f_fine = CF.pore_rhs(setup, s.plans[0].labels)
    t2 = time.time()
    p0 = s.plans[0]
    print(f"{setup.name}: levels {len(s.plans)} N_I {p0.n_internal} N_G {p0.n_ghosts} batches {[int(p.ghost_batch.max())+1 if p.n_ghosts else 0 for p in s.plans]} "
          f"hierarchy {t1-t0:.1f}s plans+upload {t2-t1:.1f}s", flush=True)
    s._set_data(s.f_fine, s.g_fine)
    s._put_u(np.zeros(p0.n_nodes))
    s.ctx.cycle(1); s.ctx.synchronize()
    s.ctx.profile(True)
    t = time.time(); s.ctx.cycle(cycles); s.ctx.synchronize(); dt = (time.time() - t) / cycles
    tot = 0
    for k in _lib.KCLASS:
        ms, n = s.ctx.profile_read(k)
        tot += ms
        print(f"   {k:12s} {ms/cycles:9.3f} ms/cycle  ({n//cycles} launches/cycle)")
    s.ctx.profile(False)
    t = time.time(); s.ctx.cycle(cycles); s.ctx.synchronize(); dt2 = (time.time() - t) / cycles
    dof = p0.n_internal + p0.n_ghosts
    print(f"   wall {dt*1e3:.2f} ms/cycle profiled, {dt2*1e3:.2f} ms/cycle plain -> {dof/dt2:.3e} DOF*cycles/s; launches {s.ctx.launches}", flush=True)
    print("   residual", s._residual_norm())

if __name__ == "__main__":
    which = sys.argv[1:] or ["c3:128"]
    for w in which:
        name, N = w.split(":")
        N = int(N)
        if name == "c4":
            probe(CF.config_pores(N=N))
        else:
            probe(CF.CONFIGS[name](N))
