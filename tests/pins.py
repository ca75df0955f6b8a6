"""Independent reference routes used to pin the oracle (test helpers; no oracle code here).

* ``intensity_mp``      Eq.(2) evaluated literally in mpmath.
* ``loglik_eq4_quad``   Eq.(4): Part1 by direct evaluation of Eq.(2) at every event,
                        Gamma = sum_i int_0^T lambda^i(v) dv by mpmath quadrature over the
                        event-free sub-intervals (the integrand is smooth there).  This does not
                        use App. B's closed form, so it pins it.
* ``ozaki_d1``          the univariate recursion of Ozaki (1979), cited at P:270.
"""
from __future__ import annotations

import mpmath
import numpy as np


def intensity_mp(theta, alpha, beta, t, mark, i, v):
    s = mpmath.mpf(theta[i])
    for tk, j in zip(t, mark):
        tk = mpmath.mpf(float(tk))
        if tk < v:
            s += mpmath.mpf(alpha[i][j]) * mpmath.exp(-mpmath.mpf(beta[i][j]) * (v - tk))
    return s


def loglik_eq4_quad(theta, alpha, beta, t, mark, T, dps=30):
    """lnL via Eq.(4): sum ln lambda - integral (quadrature).  Returns (lnl, gamma) as floats."""
    with mpmath.workdps(dps):
        D = len(theta)
        t = [float(x) for x in t]
        part1 = mpmath.mpf(0)
        for tn, i in zip(t, mark):
            part1 += mpmath.log(intensity_mp(theta, alpha, beta, t, mark, int(i), mpmath.mpf(tn)))
        knots = sorted(set([0.0, float(T)] + [x for x in t if 0.0 <= x <= T]))
        gamma = mpmath.mpf(0)
        for i in range(D):
            for a, b in zip(knots[:-1], knots[1:]):
                if b <= a:
                    continue
                # on (a, b) the set {k: t_k < v} is constant: integrate the smooth function
                gamma += mpmath.quad(lambda v: intensity_mp(theta, alpha, beta, t, mark, i, v), [a, b])
        return float(part1 - gamma), float(gamma)


def ozaki_d1(theta, alpha, beta, t, T):
    """Univariate exponential Hawkes log-likelihood via Ozaki's recursion (textbook form):
    A_1 = 0, A_n = exp(-beta (t_n - t_{n-1})) (1 + A_{n-1});
    lnL = sum_n ln(theta + alpha A_n) - theta T + (alpha/beta) sum_k (exp(-beta (T - t_k)) - 1).
    Assumes strictly increasing times."""
    A = 0.0
    s = 0.0
    prev = None
    for tn in t:
        if prev is not None:
            A = np.exp(-beta * (tn - prev)) * (1.0 + A)
        s += np.log(theta + alpha * A)
        prev = tn
    comp = sum(np.exp(-beta * (T - tk)) - 1.0 for tk in t)
    return s - theta * T + (alpha / beta) * comp
