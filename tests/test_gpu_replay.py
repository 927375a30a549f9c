"""GPU parity of the batched subdomain-local replay (osam_opinf_replay, NEXT-4) against the oracle's
regularisation selection (oracle/opinf.py select_lambda; reading R34)."""
import numpy as np
import pytest

import osam_inputs as I
from oracle import opinf

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def osam():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_20687_b200 import osam as o
    o.lib()
    return o


@pytest.fixture(scope="module")
def c2_reduced_training():
    cfg = I.config("c2")
    Xf, Xs = opinf.training_snapshots_single_domain(cfg, I)[1]
    ops = opinf.build_rom_operators(Xf, Xs, cfg["dt"], cfg["rom"]["r"], cfg["rom"]["lam"], cfg["rom"]["energy"])
    return ops["Phi"].T @ Xf, ops["Phi_s"].T @ Xs, cfg["dt"]


def _check(osam, Ubar, Ghat, dt, grid, order):
    best, errs, Os = opinf.select_lambda(Ubar, Ghat, dt, grid, order)
    g_err, g_best, traj = osam.opinf_replay(np.stack(Os), Ubar, Ghat, dt, order, trajectories=True)
    assert g_best == best
    stable = np.isfinite(errs) & (errs < 10.0)
    # errors at the rounding floor (exactly recovered operators) get an absolute floor of 1e-12
    assert np.all(np.abs(g_err[stable] - errs[stable]) <= TOL * errs[stable] + 1e-12)
    assert np.all(~np.isfinite(g_err[~stable]) | (g_err[~stable] >= 10.0))
    ref = opinf.rom_replay(Os[best], Ubar, Ghat, dt, order)
    assert np.linalg.norm(traj[best].T - ref) <= TOL * np.linalg.norm(ref)
    return errs, g_err


def test_c2_paper_grid_and_data_scale_grid(osam, c2_reduced_training):
    Ubar, Ghat, dt = c2_reduced_training
    for grid in (opinf.lambda_grid(), np.logspace(-12, -4, 40)):
        errs, g_err = _check(osam, Ubar, Ghat, dt, grid, 1)
        print("c2 grid", grid[0], grid[-1], "best err", np.nanmin(g_err))


@pytest.mark.parametrize("order", [2, 3])
def test_polynomial_candidates(osam, c2_reduced_training, order):
    Ubar, Ghat, dt = c2_reduced_training
    Ubar, Ghat = Ubar[:6], Ghat[:5]
    _check(osam, Ubar, Ghat, dt, np.logspace(-12, -2, 12), order)


def test_exact_operator_data(osam):
    rng = np.random.default_rng(5)
    r, r_b, K, dt = 4, 3, 400, 1e-3
    Kbar = np.diag([20.0, 50.0, 120.0, 300.0]) ** 2 * 1e-2
    Bbar = rng.standard_normal((r, r_b))
    t = dt * np.arange(K)
    Ghat = np.stack([np.sin(7 * t), np.cos(3 * t), t], axis=0)
    Ubar = np.zeros((r, K))
    Ubar[:, 0] = rng.standard_normal(r)
    Ubar = opinf.rom_replay(np.concatenate([-Kbar, Bbar], axis=1), Ubar, Ghat, dt)
    errs, g_err = _check(osam, Ubar, Ghat, dt, np.array([1e-14, 1e-6, 1e-2, 1.0]), 1)
    assert g_err[0] < 1e-8


def test_larger_random_models_and_velocity(osam):
    """r = 64, r_b = 40, 40 models, 600 steps, nonzero v^_0: several warps per row block, many rows per warp."""
    rng = np.random.default_rng(9)
    r, r_b, K, dt, B = 64, 40, 600, 1e-4, 40
    w = np.linspace(100.0, 15000.0, r)
    Q = np.linalg.qr(rng.standard_normal((r, r)))[0]
    base = np.concatenate([-(Q * w ** 2) @ Q.T, 10.0 * rng.standard_normal((r, r_b))], axis=1)
    Os = np.stack([base * (1.0 + 0.01 * k) for k in range(B)])
    Ghat = 1e-3 * rng.standard_normal((r_b, K))
    Ubar = 1e-3 * rng.standard_normal((r, K))
    v0 = rng.standard_normal(r) * 1e-2
    g_err, g_best, traj = osam.opinf_replay(Os, Ubar, Ghat, dt, 1, vh0=v0, trajectories=True)
    for b in (0, 17, 39):
        ref = opinf.rom_replay(Os[b], Ubar, Ghat, dt, 1, vh0=v0)
        assert np.linalg.norm(traj[b].T - ref) <= TOL * np.linalg.norm(ref)
        assert abs(g_err[b] - opinf.trajectory_error(Ubar, ref)) <= TOL * g_err[b]
