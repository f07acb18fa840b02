"""Stage-by-stage parity table of the CUDA path against the committed golden vectors
(reference outputs).  Run on the GPU box:  python scripts/gpu_stage_report.py [case ...]"""
import sys
import traceback
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from conftest import ALL_CASES, STAGED_CASES, load_golden, product_problem, product_settings, rel_inf, trace_rows  # noqa: E402

import paper_2510_07625_b200 as gb  # noqa: E402
from paper_2510_07625_b200.batch import pack_problems  # noqa: E402


def dinv_from_factor(Linv, nb, n):
    """D_k^-1 = L_k^-T L_k^-1 from the packed inverse Cholesky factors"""
    Li = np.zeros((nb, n, n))
    tri = Linv.reshape(nb, n * (n + 1) // 2)
    for i in range(n):
        for j in range(i + 1):
            Li[:, i, j] = tri[:, i * (i + 1) // 2 + j]
    return np.einsum("kli,klj->kij", Li, Li)


def stage_report(name):
    g = load_golden(name)
    problem, st = product_problem(g), product_settings(g)
    N, n, m = problem.horizon, problem.model.state_dim, problem.model.control_dim
    import dataclasses
    st1 = dataclasses.replace(st, max_sqp_iterations=1, step_tolerance=None)
    eng = gb.BatchEngine(problem.model, 1, N, problem.timestep, st1, stage_arrays=True)
    packed = pack_problems([problem], [(g["X0"], g["U0"])], [st.rho_init])
    eng.solve(packed)
    got = {k: eng.scratch(k) for k in ("A", "B", "e", "grad", "hinv", "Sdiag", "Soff", "Linv", "gamma", "lam",
                                       "dX", "dU", "merits", "pcg_iters")}
    grad = got["grad"].reshape(N + 1, n + m)
    rows = [
        ("A", got["A"].reshape(N, n, n), g["A"]), ("B", got["B"].reshape(N, n, m), g["B"]),
        ("e", got["e"].reshape(N, n), g["e"]), ("q", grad[:, :n], g["q"]), ("r", grad[:N, n:], g["r"]),
        ("q_inv0", got["hinv"][:n * n].reshape(n, n), g["q_inv"][0]),
        ("Sdiag", got["Sdiag"].reshape(N + 1, n, n), g["Sdiag"]), ("Soff", got["Soff"].reshape(N, n, n), g["Soff"]),
        ("Dinv", dinv_from_factor(got["Linv"], N + 1, n), g["Pdiag"]), ("gamma", got["gamma"], g["gamma"]),
        ("lam", got["lam"], g["lam"]), ("dX", got["dX"].reshape(N + 1, n), g["dX"]),
        ("dU", got["dU"].reshape(N, m), g["dU"]), ("merits", got["merits"][:len(g["merits"])], g["merits"]),
    ]
    line = " ".join(f"{k}={rel_inf(a, b):.1e}" for k, a, b in rows)
    print(f"{name:24s} pcg {int(got['pcg_iters'][0])}/{int(g['pcg_iterations'])} {line}", flush=True)
    eng.close()


def solve_report(name):
    g = load_golden(name)
    problem, st = product_problem(g), product_settings(g)
    res = gb.sqp_solve(problem, g["X0"], g["U0"], st)
    tr = trace_rows(res)
    ref = g["trace"]
    k = min(len(tr), len(ref))
    print(f"{name:24s} X={rel_inf(res.X, g['X']):.2e} U={rel_inf(res.U, g['U']):.2e} its {len(tr)}/{len(ref)} "
          f"conv {res.converged}/{bool(g['converged'])} pcg_gpu={tr[:k, 5].astype(int).tolist()[:8]} "
          f"pcg_ref={ref[:k, 5].astype(int).tolist()[:8]} alpha_eq={np.array_equal(np.nan_to_num(tr[:k, 3], nan=-1), np.nan_to_num(ref[:k, 3], nan=-1))} "
          f"merit_rel={rel_inf(tr[:k, 1], ref[:k, 1]):.1e}", flush=True)


if __name__ == "__main__":
    names = sys.argv[1:]
    for name in (names or STAGED_CASES):
        try:
            stage_report(name)
        except Exception:
            traceback.print_exc()
    for name in (names or ALL_CASES):
        try:
            solve_report(name)
        except Exception:
            traceback.print_exc()
