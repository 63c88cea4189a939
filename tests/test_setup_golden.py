"""The repo's own host setup against the reference's, case by case.

Every golden record holds sha256 digests of the reference's per-level plan
arrays (labels, ghost list, stencil corners, row weights, dtau, promotions,
sweep batches, band plan), produced by tests/golden/make_golden.py from the
reference's classify / SweepPlan / ExtrapolationPlan objects.  Rebuilding
each case with this package's build_hierarchy + build_level_plan must give
the same bytes: classification and ghost lists bit-exact (BASELINE.json
north star), and the plans the device consumes identical to the reference's.
"""

import pytest

import goldutil as GU

# the large cases take 10-60 s of host setup each
LARGE = {"ball256", "flowerD2048", "flowerM2048", "pores128"}
NAMES = [n for n in GU.case_names() if n in GU.CASES]


@pytest.mark.parametrize("name", [pytest.param(n, marks=pytest.mark.slow) if n in LARGE else n for n in NAMES])
def test_repo_setup_matches_reference_plans(name):
    rec = GU.record(name)
    plans, _ = GU.rebuild(name)
    assert len(plans) == rec["n_levels"]
    for lvl, p in enumerate(plans):
        got = {k: GU.plan_digest(v) for k, v in p.to_arrays().items()}
        want = rec["plan_digests"][lvl]
        bad = sorted(k for k in want if got.get(k) != want[k])
        assert not bad, (name, lvl, bad)


def test_every_golden_case_is_consumed():
    """Each reference-golden record is exercised by the oracle tests (and the
    -m gpu tests): stored plans, or a registry setup to rebuild them."""
    for n in GU.case_names():
        assert GU.has_plans(n) or n in GU.CASES, n
