"""Grasp wrench metrics (host side) against
brute-force oracles; no GPU."""
import numpy as np
import pytest


def support_min(w, rng, n_dirs=200000, refine=200):
    """min over unit u of max_i u . w_i (the support function), by dense random
    sampling then local random-perturbation refinement: an upper bound that
    converges to epsilon from above (ACCEPTANCE 4's brute-force oracle)."""
    u = rng.normal(size=(n_dirs, w.shape[1]))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    h = np.max(u @ w.T, axis=1)
    best = u[np.argsort(h)[:20]]
    out = float(np.min(h))
    for b in best:
        cur, hc = b, float(np.max(w @ b))
        step = 0.05
        for _ in range(refine):
            cand = cur + step * rng.normal(size=(64, w.shape[1]))
            cand /= np.linalg.norm(cand, axis=1, keepdims=True)
            hv = np.max(cand @ w.T, axis=1)
            k = int(np.argmin(hv))
            if hv[k] < hc:
                cur, hc = cand[k], float(hv[k])
            else:
                step *= 0.7
        out = min(out, hc)
    return out


def test_trivial_cases():
    from paper_2306_08132_b200 import metrics
    assert metrics.wrench_hull_metrics(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(3)) == (0.0, 0.0)
    e, v = metrics.wrench_hull_metrics([[1.0, 0, 0]], [[1.0, 0, 0]], np.zeros(3))
    assert e == 0.0  # one contact cannot resist pull-off
    # two antipodal contacts: no torque about their axis -> degenerate hull
    e, v = metrics.wrench_hull_metrics([[1.0, 0, 0], [-1.0, 0, 0]], [[1.0, 0, 0], [-1.0, 0, 0]], np.zeros(3))
    assert e == 0.0 and v == 0.0
    with pytest.raises(ValueError):
        metrics.wrench_hull_metrics([[1.0, 0, 0]], [[1.0, 0, 0]], np.zeros(3), cone_edges=2)


def test_epsilon_vs_support_function_oracle():
    from paper_2306_08132_b200 import metrics
    rng = np.random.default_rng(0)
    # four contacts at tetrahedron directions on a unit sphere (a force-closure grasp)
    P = np.array([[1, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]], np.float64) / np.sqrt(3.0)
    eps, vol = metrics.wrench_hull_metrics(P, P, np.zeros(3), mu=1.0, cone_edges=8)
    assert eps > 0 and vol > 0
    w = metrics.contact_wrenches(P, P, np.zeros(3), 1.0, 8)
    oracle = support_min(w, rng)
    assert oracle >= eps * (1 - 1e-9)          # the oracle is an upper bound
    assert abs(eps - oracle) / oracle < 0.01   # within 1% (SPEC ACCEPTANCE 4)


def test_epsilon_scale_invariance_and_monotone_contacts():
    from paper_2306_08132_b200 import metrics
    rng = np.random.default_rng(1)
    P = rng.normal(size=(6, 3))
    P /= np.linalg.norm(P, axis=1, keepdims=True)
    e1, _ = metrics.wrench_hull_metrics(P, P, np.zeros(3))
    e2, _ = metrics.wrench_hull_metrics(3.7 * P, P, np.zeros(3))
    assert e1 > 0 and abs(e1 - e2) < 1e-12 * max(1.0, e1)
    # more contacts (a superset) cannot shrink the hull
    Q = np.concatenate([P, rng.normal(size=(3, 3))])
    Q[6:] /= np.linalg.norm(Q[6:], axis=1, keepdims=True)
    e3, v3 = metrics.wrench_hull_metrics(Q, Q, np.zeros(3))
    _, v1 = metrics.wrench_hull_metrics(P, P, np.zeros(3))
    # lambda = 1 / r_max is unchanged (all on the unit sphere), so hulls nest
    assert e3 >= e1 - 1e-12 and v3 >= v1 - 1e-12


def test_sweep_and_topk(tmp_path):
    from paper_2306_08132_b200 import metrics
    reps = [[dict(threshold_mm=t, contact_area_cm2=t * (k + 1), contacts=int(t), epsilon=0.01 * k, gws_volume=0.1 * t)
             for t in (1.0, 2.0, 5.0)] for k in range(20)]
    rows = metrics.threshold_sweep(reps, str(tmp_path / "s.csv"))
    assert [r["threshold_mm"] for r in rows] == [1.0, 2.0, 5.0]
    assert rows[0]["mean_CA_cm2"] <= rows[1]["mean_CA_cm2"] <= rows[2]["mean_CA_cm2"]
    txt = (tmp_path / "s.csv").read_text().splitlines()
    assert txt[0] == "threshold_mm,mean_CA_cm2,mean_eps,mean_vol" and len(txt) == 4
    assert metrics.top_k(reps, 10) == list(range(19, 9, -1))
