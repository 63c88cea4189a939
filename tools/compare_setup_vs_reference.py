import sys, time, math
import numpy as np
sys.path.insert(0, '/root/reference/pkg/src')
import ghostmg.geometry as RG, ghostmg.transfer as RT, ghostmg.operators as RO, ghostmg.smoothing as RS, ghostmg.levelsets as RL, ghostmg.cases as RC
from ghostmg.smoothing import SmootherConfig as RSC
import paper_2207_14208_b200.geometry as G, paper_2207_14208_b200.transfer as T, paper_2207_14208_b200.operators as O
import paper_2207_14208_b200.smoothing as S, paper_2207_14208_b200.levelsets as L

def beq(a, b, name):
    a = np.asarray(a); b = np.asarray(b)
    ok = a.shape == b.shape and (np.array_equal(a.view(np.uint8), b.view(np.uint8)) if a.dtype == b.dtype else False)
    if not ok:
        print('MISMATCH', name, a.shape, b.shape, a.dtype, b.dtype)
        if a.shape == b.shape and a.dtype.kind == 'f':
            print('  maxdiff', np.nanmax(np.abs(a - b)))
    return ok

def compare(name, d, N, phi, faces=(), bc='dirichlet', variant='exp', coarsest_min=4):
    t = time.time()
    rl = RT.build_hierarchy(RG.UniformGrid(d, N), phi, faces, coarsest_min=coarsest_min)
    t1 = time.time()
    ml = T.build_hierarchy(G.UniformGrid(d, N), phi, faces, coarsest_min=coarsest_min)
    t2 = time.time()
    ok = len(rl) == len(ml)
    for li, (r, m) in enumerate(zip(rl, ml)):
        rc, mc = r.cls, m.cls
        for f in ['labels', 'ghost_idx', 'ghost_Q', 'ghost_n', 'ghost_theta', 'ghost_theta_raw', 'ghost_stencil', 'ghost_block_low', 'ghost_promoted', 'internal_idx', 'eliminated_idx', 'inactive_idx']:
            ok &= beq(getattr(rc, f), getattr(mc, f), f'{name} L{li} {f}')
        rw = RO.ghost_row_weights(rc, bc); mw = O.ghost_row_weights(mc, bc)
        ok &= beq(rw, mw, f'{name} L{li} weights')
        rd = RS.assign_dtau(rc, bc, RSC(), variant); md = S.assign_dtau(mc, bc, S.SmootherConfig(), variant)
        ok &= beq(rd, md, f'{name} L{li} dtau')
        re, me = r.extrap, m.extrap
        ok &= len(re.bfs_groups) == len(me.bfs_groups)
        for gi, ((ri, rn, rm), (mi, mm)) in enumerate(zip(re.bfs_groups, me.bfs_groups)):
            ok &= beq(ri, mi, f'bfs idx {gi}')
            bits = np.zeros(len(ri), np.uint8)
            for c in range(rm.shape[1]): bits |= rm[:, c].astype(np.uint8) << c
            ok &= beq(bits, mm, f'bfs mask {gi}')
        ok &= beq(re.band_idx, me.band_idx, 'band')
        ok &= beq(re.trans_nbrs, me.neighbours(mc.grid.strides), 'trans nbrs')
        ok &= beq(re.trans_absn, me.trans_absn, 'trans absn')
    print(name, 'levels', len(rl), 'ok' if ok else 'FAIL', f'ref {t1-t:.2f}s mine {t2-t1:.2f}s', [l.cls.n_ghosts for l in ml])
    return ok

compare('disk64', 2, 64, L.SignedSphere((0.02, 0.01), 0.5))
compare('disk256', 2, 256, L.SignedSphere((0.02, 0.01), 0.5))
compare('circle32', 2, 32, RL.Sphere((math.sqrt(3)/40, -0.05), math.sqrt(2)/2))
compare('flower128N', 2, 128, RL.Flower(0.5, 0.15), bc='neumann', coarsest_min=32)
compare('flower128D', 2, 128, L.Flower(0.5, 0.2))
compare('sphere32', 3, 32, L.SignedSphere((0.013, -0.007, 0.021), 0.45), coarsest_min=8)
compare('sphere64', 3, 64, L.SignedSphere((0.013, -0.007, 0.021), 0.45), coarsest_min=8)
compare('ellipsoid32', 3, 32, RL.Ellipsoid((math.sqrt(2)/20, math.sqrt(3)/40, -math.sqrt(2)/50), (0.686, 0.386, 0.586)))
cs = RC.build_case('vline', 64, 0.5); compare('vline64', 2, 64, cs.phi, cs.eliminated_faces, variant='poly')
cs = RC.build_case('plane3d', 16, 0.5); compare('plane3d16', 3, 16, cs.phi, cs.eliminated_faces, variant='poly')
cs = RC.build_case('line30', 32, 0.5); compare('line30', 2, 32, cs.phi, cs.eliminated_faces, bc='neumann')
pore = L.pore_space_unit_cube(42, 64, 0.05, 0.15)
faces = [(a, s) for a in range(3) for s in (0, 1)]
compare('pores64', 3, 64, pore, faces, bc='neumann', coarsest_min=4)
