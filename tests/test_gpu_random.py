"""GPU parity on randomly STRUCTURED systems: every engine (grid, cluster,
batch) against the oracle, bit for bit, over systems the pinned configs do
not cover -- ragged equations (1 to 14 terms), exponents 1-4 (the exponent
pass of the reverse mode), constant terms, repeated monomials
across equations (the deduplicated table), variables absent
from whole equations (structural Jacobian zeros) and DD / QD coefficients
with every limb populated (the hi-only stream selection of the batch,
DESIGN.md §5.2, must not fire on them).  Whatever a path does -- converge,
fail at the start, stall at h_min, run out of steps -- the stats, the trace
and the end point must be identical to the oracle's.
"""
import numpy as np
import pytest

from conftest import assert_bits_equal

import paper_1501_06625_b200 as pt
from paper_1501_06625_b200 import PrecisionMode as PM
from structured import CASES, case, max_steps

pytestmark = pytest.mark.gpu


def compare(out, end, st, tr):
    assert out.success == (st.status == 0)
    assert (out.steps, out.accepted, out.newton_iters, out.start_iters) == (
        st.steps, st.accepted, st.newton_iters, st.start_iters)
    assert_bits_equal(np.array([out.final_residual, out.final_update, out.t_end]),
                      np.array([st.final_residual, st.final_update, st.t_end]), "stats")
    if tr is not None:
        assert len(out.trace) == len(tr)
        for a, b in zip(out.trace, tr):
            assert (a.ok, a.iters) == (b.ok, b.iters)
            assert_bits_equal(np.array([a.t, a.residual, a.update]), np.array([b.t, b.residual, b.update]), "trace")
    assert_bits_equal(out.end, end, "end point")


@pytest.mark.parametrize("n,prec,seed", CASES, ids=lambda v: str(v) if not isinstance(v, PM) else v.name)
def test_random_structure_single_path_engines(gpu, oracle, n, prec, seed):
    f, g, gamma, params, starts = case(n, prec, seed, max_steps(prec))
    cap = params.max_steps + 2
    hom = pt.make_homotopy(g, f, gamma, 2, device=gpu)
    for p in range(2):
        end, st, tr = oracle.track_path(int(prec), g, f, gamma, 2, starts[p], params, cap)
        for engine in ("grid", "cluster"):
            hom.set_engine(engine)
            compare(hom.track_path(starts[p], params, trace=True), end, st, tr)


@pytest.mark.parametrize("n,prec,seed", CASES, ids=lambda v: str(v) if not isinstance(v, PM) else v.name)
def test_random_structure_batch(gpu, oracle, n, prec, seed):
    f, g, gamma, params, starts = case(n, prec, seed, max_steps(prec))
    hom = pt.make_homotopy(g, f, gamma, 2, device=gpu)
    ends, outs = hom.track_batch(starts, params)
    for p in range(starts.shape[0]):
        end, st, _ = oracle.track_path(int(prec), g, f, gamma, 2, starts[p], params)
        compare(outs[p], end, st, None)
        assert_bits_equal(ends[p], end, f"batch path {p}")
