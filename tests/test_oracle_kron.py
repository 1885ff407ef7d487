"""Pin the matrix-free Kronecker oracle (oracle/kron.py, the checker of the 256^3 / 512^3
GPU tests) to the 3D-assembled oracle and to the reference's own golden vectors."""

import numpy as np
import pytest

from oracle import kron
from oracle import problems as op
from oracle import solvers as so


@pytest.mark.parametrize("spec,n,m0", [
    (op.thermal_block((2, 1, 1)), 8, 2),
    (op.thermal_block((2, 2, 1)), 16, 4),
    (op.thermal_block((2, 2, 2)), 16, 4),
    (op.smooth_affine(6), 16, 4),
])
def test_operators_match_3d_assembly(spec, n, m0):
    P, K = op.OracleProblem(spec, n, m0), kron.KronProblem(spec, n, m0)
    mu = op.sample_mus(spec, 1, seed=3)[0]
    for lvl in range(P.levels):
        A = P.operator(mu, lvl).toarray()
        if lvl == 0:
            B = K.dense(mu, 0)
        else:
            S = K.stencil(mu, lvl)
            B = np.column_stack([S @ e for e in np.eye(A.shape[0])])
        assert np.max(np.abs(A - B)) <= 1e-14 * np.max(np.abs(A)), lvl
    np.testing.assert_array_equal(K.rhs(), P.rhs())


def test_plane_windows_match_whole_level():
    spec = op.smooth_affine(6)
    K = kron.KronProblem(spec, 16, 4)
    mu = op.sample_mus(spec, 1, seed=8)[0]
    x = np.random.default_rng(1).standard_normal(15 ** 3)
    full = (K.stencil(mu) @ x).reshape(15, 15, 15)
    xp = np.zeros((17, 17, 17))
    xp[1:-1, 1:-1, 1:-1] = x.reshape(15, 15, 15)
    for k0, k1 in [(0, 4), (6, 9), (12, 15)]:
        y = K.stencil(mu, k0=k0, k1=k1).apply_planes(xp[k0:k1 + 2])
        np.testing.assert_allclose(y, full[k0:k1], rtol=0, atol=1e-15 * np.abs(full).max())


def test_vcycle_and_mgcg_match_reference_golden(golden):
    K = kron.KronProblem(op.thermal_block((2, 2, 1)), 16, 4)
    out = so.mg_vcycle(golden["vcycle_tb221_n16_in"], kron.mg_context_for(K, golden["vcycle_tb221_n16_mu"]))
    ref = golden["vcycle_tb221_n16_out"]
    assert np.linalg.norm(out - ref) <= 1e-13 * np.linalg.norm(ref)
    for tag, spec, n in [("tb221", op.thermal_block((2, 2, 1)), 32),
                         ("smooth6", op.smooth_affine(6), 16)]:
        K = kron.KronProblem(spec, n, 4)
        key = f"mgcg_{tag}_n{n}"
        delta = float(golden[key + "_delta"])
        for m, xr, it in zip(golden[key + "_mus"], golden[key + "_x"], golden[key + "_iters"]):
            x, rep = kron.mgcg_solve(K, m, delta=delta, l_max=60)
            assert rep.iterations == it
            assert np.linalg.norm(x - xr) <= 1e-10 * np.linalg.norm(xr)
