"""Pins of the GSC-Falkon / LogFalkon oracle (Alg. 2), -m "not gpu".

None re-types the oracle's formulas: losses against golden values and
finite differences; the step against Alg. 1 (oracle.fit, a different code path) through two
exact reductions; against the dense Newton step (explicit Hessian and gradient, numpy solve);
against scipy.optimize on the objective alone; and symmetry / monotonicity properties.
"""
import math
import os

import numpy as np
import pytest
import scipy.optimize as so

import oracle
from oracle import gsc

GOLD = os.path.join(os.path.dirname(__file__), "golden")
G = oracle.GAUSSIAN


def _problem(n=60, m=8, d=3, seed=0, sigma=1.3, labels="pm1"):
    r = np.random.default_rng(seed)
    X = r.standard_normal((n, d)).astype(np.float32).astype(np.float64)
    idx = r.choice(n, m, replace=False)
    C = X[idx]
    f = np.sin(X[:, 0] + X[:, 1]) + 0.3 * r.standard_normal(n)
    y = np.where(f >= 0, 1.0, -1.0) if labels == "pm1" else f
    return X, y, C, y[idx], sigma


def _golden_losses():
    rows = []
    with open(os.path.join(GOLD, "gsc_losses.txt")) as fh:
        for line in fh:
            if line.startswith("#") or not line.strip():
                continue
            p = line.split()
            rows.append((p[0], p[1], float(p[2]), float(p[3]), float(p[4])))
    return rows


@pytest.mark.parametrize("row", _golden_losses())
def test_loss_golden(row):
    """tests/golden/gsc_losses.txt: analytic values of the logistic loss (SPEC.md:390-391,
    Example 1(a) PAPER.md:1026) and of the squared loss."""
    kind, what, z, y, expected = row
    k = gsc.LOGISTIC if kind == "logistic" else gsc.SQUARED
    val, d1, d2 = gsc.loss_eval(k, np.array([z]), np.array([y]))
    got = {"value": val, "d1": d1, "d2": d2}[what][0]
    assert abs(got - expected) <= 1e-12 * max(1.0, abs(expected))


@pytest.mark.parametrize("kind", [gsc.LOGISTIC, gsc.SQUARED])
def test_loss_derivatives_finite_differences(kind):
    """l' and l'' match central differences of l (Def. 1: three times differentiable)."""
    r = np.random.default_rng(1)
    z = r.uniform(-6, 6, 200)
    y = np.where(r.random(200) < 0.5, -1.0, 1.0)
    h = 1e-4
    v = lambda zz: gsc.loss_eval(kind, zz, y)[0]
    d1 = lambda zz: gsc.loss_eval(kind, zz, y)[1]
    _, g, H = gsc.loss_eval(kind, z, y)
    assert np.max(np.abs(g - (v(z + h) - v(z - h)) / (2 * h))) < 1e-7
    assert np.max(np.abs(H - (d1(z + h) - d1(z - h)) / (2 * h))) < 1e-7
    assert np.all(H >= 0)  # convexity (Def. 1)


def test_logistic_loss_no_overflow():
    val, d1, d2 = gsc.loss_eval(gsc.LOGISTIC, np.array([800.0, -800.0]), np.array([1.0, 1.0]))
    assert np.all(np.isfinite(val)) and abs(val[1] - 800.0) < 1e-9 and val[0] == 0.0
    assert np.all(np.isfinite(d1)) and np.all(np.isfinite(d2))


def test_squared_loss_reduces_to_falkon():
    """Reading g3: with l = (z - y)^2/2 (D = I, g = z - y) one GSC step from alpha = 0 is
    exactly Alg. 1 (oracle.fit): same preconditioner, R = P^T Knm^T y, same LinOp."""
    X, y, C, yC, s = _problem(labels="real")
    lam, t = 1e-3, 6
    a_gsc = gsc.gsc_falkon(X, y, C, yC, gsc.SQUARED, G, s, [lam], [t])
    a_fal = oracle.fit(X, y, C, G, s, lam, t)
    assert np.linalg.norm(a_gsc - a_fal) <= 1e-9 * np.linalg.norm(a_fal)


def test_first_logistic_step_is_scaled_falkon():
    """At alpha = 0: z = 0, D = I/4, g = -y/2, so the Newton system is
    (Knm^T Knm + 4 mu n K) alpha = 2 Knm^T y and the weighted preconditioner is
    (1/2) x Falkon's at lambda = 4 mu; CG is invariant to that scaling, hence the first step
    equals oracle.fit(X, 2y, C, 4 mu, t) for every t."""
    X, y, C, yC, s = _problem()
    mu = 2e-3
    for t in (1, 3, 7):
        a = gsc.weighted_falkon(X, y, C, yC, gsc.LOGISTIC, G, s, mu, t, np.zeros(len(C)))
        b = oracle.fit(X, 2.0 * y, C, G, s, 4.0 * mu, t)
        assert np.linalg.norm(a - b) <= 1e-9 * np.linalg.norm(b), t


def _dense_newton(X, y, C, alpha, mu, s, jitter=oracle.DEFAULT_JITTER):
    """Textbook Newton step on J(alpha) = mean l(Knm alpha) + mu/2 alpha^T K alpha, built from
    explicit matrices (brute-force kernel, not the oracle's products)."""
    Knm = np.array([[math.exp(-np.sum((x - c) ** 2) / (2 * s * s)) for c in C] for x in X])
    K = np.array([[math.exp(-np.sum((a - b) ** 2) / (2 * s * s)) for b in C] for a in C])
    K = K + jitter * np.eye(len(C))
    n = len(X)
    z = Knm @ alpha
    p = 1.0 / (1.0 + np.exp(-y * z))          # sigma(y z)
    g = -y * (1.0 - p)
    D = p * (1.0 - p)
    grad = Knm.T @ g / n + mu * K @ alpha
    H = Knm.T @ (D[:, None] * Knm) / n + mu * K
    return alpha - np.linalg.solve(H, grad), Knm, K


def test_step_with_converged_cg_is_the_newton_step():
    """t >= m: the preconditioned CG solves the step's system exactly, so WeightedFalkon from
    any alpha_0 equals the dense Newton step alpha_0 - H^-1 grad J (PAPER.md:1051-1053,
    readings g1-g4, g6)."""
    X, y, C, yC, s = _problem(m=10)
    r = np.random.default_rng(5)
    a0 = 0.3 * r.standard_normal(len(C))
    mu = 1e-2
    got = gsc.weighted_falkon(X, y, C, yC, gsc.LOGISTIC, G, s, mu, 40, a0)
    want, _, _ = _dense_newton(X, y, C, a0, mu, s)
    assert np.linalg.norm(got - want) <= 1e-7 * np.linalg.norm(want)


def test_newton_iterates_converge_to_scipy_minimiser():
    """Repeated steps at a fixed level converge to the minimiser of J, found independently by
    scipy.optimize (BFGS on the objective value alone, numerical gradients)."""
    X, y, C, yC, s = _problem(m=6, n=50)
    mu = 5e-2
    a = np.zeros(len(C))
    for _ in range(8):
        a = gsc.weighted_falkon(X, y, C, yC, gsc.LOGISTIC, G, s, mu, 20, a)
    _, Knm, K = _dense_newton(X, y, C, a, mu, s)

    def J(al):
        z = Knm @ al
        return np.mean(np.logaddexp(0.0, -y * z)) + 0.5 * mu * al @ K @ al
    res = so.minimize(J, np.zeros(len(C)), method="BFGS", options={"gtol": 1e-11})
    assert np.linalg.norm(a - res.x) <= 1e-4 * np.linalg.norm(res.x)
    assert abs(gsc.objective(X, y, C, a, gsc.LOGISTIC, G, s, mu) - J(a)) < 1e-12


def test_label_negation_negates_alpha():
    """l(z, -y) = l(-z, y): flipping every label flips the whole Newton path's alpha."""
    X, y, C, yC, s = _problem()
    mus, its = [1e-1, 1e-2, 1e-3], [3, 3, 5]
    a = gsc.gsc_falkon(X, y, C, yC, gsc.LOGISTIC, G, s, mus, its)
    b = gsc.gsc_falkon(X, -y, C, -yC, gsc.LOGISTIC, G, s, mus, its)
    assert np.linalg.norm(a + b) <= 1e-10 * np.linalg.norm(a)


def test_weighted_preconditioner_identities():
    """T^T T = Kmm + delta I; A^T A = (1/m) T D T^T + mu I with D = l''(Kmm alpha, y_m)
    (PAPER.md:996-1005), D formed here from explicit products; D = I reduces to Alg. 1's
    preconditioner at lambda = mu."""
    X, y, C, yC, s = _problem(m=12)
    r = np.random.default_rng(3)
    a = r.standard_normal(len(C))
    mu = 1e-3
    T, A, z = gsc.weighted_preconditioner(C, yC, a, gsc.LOGISTIC, G, s, mu)
    K = oracle.kmm(C, G, s)
    assert np.allclose(z, K @ a, rtol=0, atol=1e-13)
    p = 1.0 / (1.0 + np.exp(-yC * z))
    M = T @ np.diag(p * (1 - p)) @ T.T / len(C) + mu * np.eye(len(C))
    assert np.linalg.norm(A.T @ A - M) <= 1e-13 * np.linalg.norm(M)
    assert np.linalg.norm(T.T @ T - K - oracle.DEFAULT_JITTER * np.eye(len(C))) <= 1e-13 * np.linalg.norm(K)
    T2, A2, _ = gsc.weighted_preconditioner(C, yC, a, gsc.SQUARED, G, s, mu)
    T1, A1 = oracle.preconditioner(C, G, s, mu)
    assert np.allclose(T2, T1, rtol=0, atol=1e-14) and np.allclose(A2, A1, rtol=0, atol=1e-14)


def test_path_decreases_objective_and_newton_path_schedule():
    """Along Alg. 2's path the objective at the FINAL level decreases step by step on this
    well-conditioned problem; newton_path gives ceil(log(mu0/lam)/log(1/q)) + 1 levels plus
    the final one (reading g5)."""
    mus, its = gsc.newton_path(1.0, 0.1, 1e-3, 4, 8)
    assert mus == pytest.approx([1.0, 0.1, 0.01, 1e-3, 1e-3]) and its == [4, 4, 4, 4, 8]
    mus2, _ = gsc.newton_path(1.0, 0.5, 0.3, 2, 3)   # 1, .5 then .25 < .3 -> stop; final .3
    assert mus2 == pytest.approx([1.0, 0.5, 0.3])
    X, y, C, yC, s = _problem(n=80, m=10)
    mus, its = gsc.newton_path(1.0, 0.2, 1e-2, 10, 10)
    _, path = gsc.gsc_falkon(X, y, C, yC, gsc.LOGISTIC, G, s, mus, its, return_path=True)
    lam = mus[-1]
    objs = [gsc.objective(X, y, C, a, gsc.LOGISTIC, G, s, lam) for a in path]
    assert objs[-1] <= min(objs[:-1]) + 1e-12
    assert objs[0] < gsc.objective(X, y, C, np.zeros(len(C)), gsc.LOGISTIC, G, s, lam)


def test_center_labels_are_the_rows_labels():
    """synth.gen_y_rows on the centre indices equals the labels of those rows (y_m of Alg. 2,
    PAPER.md:964: the Nystrom points keep their own labels)."""
    import synth
    X = synth.gen_X(3, 0, 1000, 28)
    y = synth.gen_y(3, X, 0, "cls")
    idx = synth.center_indices(3, 1000, 50)
    assert np.array_equal(synth.gen_y_rows(3, X[idx], idx, "cls"), y[idx])
    g, Xg, yg, C, yC = synth.make_gsc_problem("tiny_log")
    idx = synth.center_indices(0, 2000, 100)
    assert np.array_equal(C, Xg[idx]) and np.array_equal(yC, yg[idx])
