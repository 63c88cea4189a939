"""z-slab sharded cycles on the device: two rank threads,
each with its own context on the one GPU of the test box, exchange planes
through queues (paper_2207_14208_b200.slabs.LocalGroup -- the interface
torch.distributed/NCCL gets in bench.py --gpus N) and must reproduce the
single-context solve bit for bit: residual history, rho and the iterate.
The kernels of the two ranks never wait on one another (every exchange is a
host-side blocking receive), so running them on one GPU is safe.
"""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(N):
    from paper_2207_14208_b200 import configs as CF
    from paper_2207_14208_b200.cycle import CycleDriver
    from paper_2207_14208_b200.transfer import build_hierarchy

    setup = CF.config_pores(N=N)
    levels = build_hierarchy(setup.grid, setup.phi, setup.faces, max_levels=setup.cycle.max_levels,
                             coarsest_min=setup.coarsest_min)
    plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
    f = CF.pore_rhs(setup, plans[0].labels)
    return setup, plans, f, g, e


@pytest.mark.parametrize("N,world", [(64, 2), (128, 2), (128, 3)])
def test_slab_solve_matches_single_context(N, world, gpu_available):
    from paper_2207_14208_b200.slabs import LocalGroup, SlabPartition, slab_solver
    from paper_2207_14208_b200.solver import MultigridSolver

    setup, plans, f, g, e = _setup(N)
    cycles = 4
    ref = MultigridSolver.from_plans(plans, f, g, e, setup.smoother, setup.cycle, coarse_backend="superlu")
    u_ref, rep_ref = ref.solve(u=np.zeros(plans[0].n_nodes), cycles=cycles)
    ref.ctx.close()

    part = SlabPartition([p.N for p in plans], world, min_N=64)
    assert part.distributed(0)
    shared = LocalGroup.Shared(world)
    out = [None] * world
    err = []

    def run(rank):
        try:
            grp = LocalGroup(shared, rank)
            s = slab_solver(plans, f, g, e, setup.smoother, setup.cycle, grp, coarse_backend="superlu")
            u, rep = s.solve(u=np.zeros(plans[0].n_nodes), cycles=cycles)
            out[rank] = (u, rep)
            s.ctx.close()
        except BaseException as exc:  # noqa: BLE001 -- reported by the main thread
            err.append((rank, exc))
            raise

    threads = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=900)
    assert not err, err
    assert all(o is not None for o in out), "a rank did not finish"
    for rank, (u, rep) in enumerate(out):
        assert rep.residual_norms == rep_ref.residual_norms, (rank, rep.residual_norms, rep_ref.residual_norms)
        assert np.array_equal(u, u_ref), rank
