"""Stage-by-stage parity of the CUDA path (through the C ABI) against the reference's golden
vectors: linearize -> Schur -> D^-1 -> PCG -> recover -> candidate merits of the first SQP
iteration.  Tolerances are relative-inf (oracles.relative_inf_error, oracles.py:166-168)."""

import dataclasses

import numpy as np
import pytest

import paper_2510_07625_b200 as gb
from paper_2510_07625_b200.batch import pack_problems
from conftest import STAGED_CASES, load_golden, product_problem, product_settings, rel_inf

pytestmark = pytest.mark.gpu


def unpack_lower(T, nb, n):
    """packed lower-triangular blocks [nb, n(n+1)/2] -> [nb, n, n] with zeros above the diagonal"""
    out = np.zeros((nb, n, n))
    tri = T.reshape(nb, n * (n + 1) // 2)
    for i in range(n):
        for j in range(i + 1):
            out[:, i, j] = tri[:, i * (i + 1) // 2 + j]
    return out


def dinv_from_factor(Linv, nb, n):
    """D_k^-1 = S_kk^-1 = L_k^-T L_k^-1 from the device's inverse Cholesky factors"""
    Li = unpack_lower(Linv, nb, n)
    return np.einsum("kli,klj->kij", Li, Li)


def pad_stride(v):
    m = (v + 1) & ~1
    return m + 2 if (m // 2) % 2 == 0 else m


@pytest.mark.parametrize("name", STAGED_CASES)
def test_first_iteration_stages_match_reference(name):
    g = load_golden(name)
    problem, st = product_problem(g), product_settings(g)
    N, n, m = problem.horizon, problem.model.state_dim, problem.model.control_dim
    one = dataclasses.replace(st, max_sqp_iterations=1, step_tolerance=None)
    eng = gb.BatchEngine(problem.model, 1, N, problem.timestep, one, stage_arrays=True)
    try:
        eng.solve(pack_problems([problem], [(g["X0"], g["U0"])], [st.rho_init]))
        got = {k: eng.scratch(k) for k in ("A", "B", "e", "grad", "hinv", "Sdiag", "Soff", "Linv", "Lfac", "gamma", "gammaw",
                                           "pmats", "lam",
                                           "dX", "dU", "merits", "pcg_iters")}
    finally:
        eng.close()
    grad = got["grad"].reshape(N + 1, n + m)
    checks = [
        ("A", got["A"].reshape(N, n, n), g["A"], 1e-11), ("B", got["B"].reshape(N, n, m), g["B"], 1e-11),
        ("e", got["e"].reshape(N, n), g["e"], 1e-11), ("q", grad[:, :n], g["q"], 1e-12),
        ("r", grad[:N, n:], g["r"], 1e-12),
        ("Q^-1", got["hinv"][:n * n].reshape(n, n), g["q_inv"][0], 1e-11),
        ("QN^-1", got["hinv"][n * n:2 * n * n].reshape(n, n), g["q_inv"][-1], 1e-11),
        ("R^-1", got["hinv"][2 * n * n:2 * n * n + m * m].reshape(m, m), g["r_inv"][0], 1e-11),
        ("S diag", got["Sdiag"].reshape(N + 1, n, n), g["Sdiag"], 1e-11),
        ("S offdiag", got["Soff"].reshape(N, n, n), g["Soff"], 1e-11),
        ("D^-1", dinv_from_factor(got["Linv"], N + 1, n), g["Pdiag"], 1e-9),
        ("gamma", got["gamma"], g["gamma"], 1e-11), ("lambda", got["lam"], g["lam"], 1e-8),
        ("dX", got["dX"].reshape(N + 1, n), g["dX"], 1e-7), ("dU", got["dU"].reshape(N, m), g["dU"], 1e-7),
        ("merits", got["merits"][:len(g["merits"])], g["merits"], 1e-8),
    ]
    for label, a, b, tol in checks:
        assert rel_inf(a, b) <= tol, f"{label}: {rel_inf(a, b):.3e} > {tol}"
    assert abs(int(got["pcg_iters"][0]) - int(g["pcg_iterations"])) <= 1
    # the whitened quantities k_schur hands to the PCG kernels (pcg_kernels.cuh)
    Lf, Li = unpack_lower(got["Lfac"], N + 1, n), unpack_lower(got["Linv"], N + 1, n)
    assert rel_inf(Lf @ Lf.transpose(0, 2, 1), g["Sdiag"]) <= 1e-11
    assert rel_inf(Li @ Lf, np.broadcast_to(np.eye(n), Lf.shape)) <= 1e-9
    assert rel_inf(got["gammaw"].reshape(N + 1, n), np.einsum("kij,kj->ki", Li, g["gamma"].reshape(N + 1, n))) <= 1e-10
    bsp, trp = pad_stride(n * n), pad_stride(n * (n + 1) // 2)
    W = got["pmats"][:N * bsp].reshape(N, bsp)[:, :n * n].reshape(N, n, n)
    assert rel_inf(W, Li[1:] @ g["Soff"]) <= 1e-10
    rec_inv = got["pmats"][N * bsp:N * bsp + (N + 1) * trp].reshape(N + 1, trp)[:, :n * (n + 1) // 2]
    assert np.array_equal(rec_inv.ravel(), got["Linv"])


@pytest.mark.parametrize("name", ["twolink_n8", "iiwa14_reach_n8_b0"])
def test_whitened_preconditioner_equals_explicit_stair_blocks(name):
    """The PCG kernels apply Phi^-1 as L^-T (I - O^) L^-1 instead of forming -D_{k+1}^-1 phi_k D_k^-1
    (qpform.py:355-356): the explicit blocks rebuilt from the device factors and phi must equal the
    reference's."""
    g = load_golden(name)
    problem, st = product_problem(g), product_settings(g)
    N, n = problem.horizon, problem.model.state_dim
    one = dataclasses.replace(st, max_sqp_iterations=1, step_tolerance=None)
    eng = gb.BatchEngine(problem.model, 1, N, problem.timestep, one, stage_arrays=True)
    try:
        eng.solve(pack_problems([problem], [(g["X0"], g["U0"])], [st.rho_init]))
        D = dinv_from_factor(eng.scratch("Linv"), N + 1, n)
        off = eng.scratch("Soff").reshape(N, n, n)
    finally:
        eng.close()
    explicit = np.stack([-D[k + 1] @ off[k] @ D[k] for k in range(N)])
    assert rel_inf(explicit, g["Poff"]) <= 1e-9


@pytest.mark.parametrize("name", ["cartpole_n8", "iiwa14_reach_n8_b0", "twolink_profile_n8"])
def test_first_iteration_stages_in_the_reference_types(name):
    """first_iteration_stages: the reference's linearize -> form_schur -> form_preconditioner -> pcg ->
    recover_step -> merit_many chain as reference-typed objects, against the golden stages."""
    g = load_golden(name)
    problem, st = product_problem(g), product_settings(g)
    N, n, m = problem.horizon, problem.model.state_dim, problem.model.control_dim
    d = gb.first_iteration_stages(problem, g["X0"], g["U0"], st)
    assert len(d.blocks) == N + 1 and d.blocks[-1].A is None and d.blocks[-1].R is None
    assert rel_inf(np.stack([b.A for b in d.blocks[:-1]]), g["A"]) <= 1e-11
    assert rel_inf(np.stack([b.q for b in d.blocks]), g["q"]) <= 1e-12
    assert np.array_equal(d.blocks[0].Q, g["Q"] + st.rho_init * np.eye(n))     # damped Hessian, undamped gradient
    assert rel_inf(d.system.S.diag_blocks, g["Sdiag"]) <= 1e-11 and rel_inf(d.system.phi, g["Soff"]) <= 1e-11
    assert rel_inf(d.system.gamma, g["gamma"]) <= 1e-11 and rel_inf(d.system.q_inv, g["q_inv"]) <= 1e-11
    assert rel_inf(d.system.phi_inv.diag_blocks, g["Pdiag"]) <= 1e-9
    assert rel_inf(d.system.phi_inv.offdiag_blocks, g["Poff"]) <= 1e-9
    assert abs(d.pcg.iterations - int(g["pcg_iterations"])) <= 1 and d.pcg.converged == bool(g["pcg_converged"])
    assert rel_inf(d.pcg.solution, g["lam"]) <= 1e-8
    assert rel_inf(d.direction.dX, g["dX"]) <= 1e-7 and abs(d.direction.inf_norm - float(g["step_inf"])) <= 1e-7
    assert rel_inf(d.merits, g["merits"]) <= 1e-8 and abs(d.merit0 - float(g["merit0"])) <= 1e-9 * abs(float(g["merit0"]))
