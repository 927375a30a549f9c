"""Oracle: closed-form 1D wave solution used as a pin (TEST INFRASTRUCTURE ONLY).

P:L839-844 eq:disp_exact gives the method-of-characteristics solution of the clamped bar;
the printed fourth term is missing its `f`. Reading R28 uses the equivalent
d'Alembert form  u(x,t) = 1/2 [F(x - ct) + F(x + ct)],  F the odd, 2L-periodic extension
of f about the clamped ends x = 0 and x = L; c = sqrt(E/rho).
"""
from __future__ import annotations

import numpy as np


def odd_periodic_extension(f, L):
    def F(x):
        y = np.mod(np.asarray(x, dtype=np.float64), 2 * L)
        return np.where(y <= L, f(np.minimum(y, L)), -f(np.clip(2 * L - y, 0, L)))
    return F


def dalembert(f, L, c, x, t):
    F = odd_periodic_extension(f, L)
    return 0.5 * (F(x - c * t) + F(x + c * t))
