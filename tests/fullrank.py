"""Full-rank "ROMs" with intrusive operators (TEST INFRASTRUCTURE): Phi = I on the free DOFs, Phi_dS = I on
the Schwarz DOFs, Kbar = M^-1 K_ff, Bbar = -M^-1 K_fs (the OpInf limit the paper's inference
recovers).  With them a ROM step is exactly the FOM step of its box, so a conformal coupled run with ROM
subdomains must equal the monolithic FOM on the union of the boxes -- an end-to-end pin for the FOM-ROM and
ROM-ROM coupling paths (per sample with the modulus scale e_b = E_b / E for batched ROMs, reading R22)."""
import copy

import numpy as np

import osam_inputs as I
from oracle import fem, schwarz


def conformal_cfg(kinds=("fom", "rom"), batch=None):
    """c1 geometry made conformal (h = 0.02 in both boxes), kinds per box, optional batch of moduli."""
    cfg = copy.deepcopy(I.config("c1"))
    cfg["subdomains"][1] = dict(cfg["subdomains"][1], nel=(30, 5, 5))
    for s, k in zip(cfg["subdomains"], kinds):
        s["kind"] = k
    cfg["dt"] = 0.5 * 0.02 / fem.p_wave_speed(I.E0 * (1.2 if batch else 1.0), I.NU, I.RHO)
    cfg["max_iters"], cfg["min_iters"] = 50, 2
    if batch:
        cfg["batch"] = len(batch)
        cfg["samples"] = dict(E=tuple(I.E0 * e for e in batch), A=tuple(1e-3 for _ in batch))
    return cfg


def full_rank_ops(cfg):
    """Intrusive operators for every ROM box of cfg (built from the oracle's FOM of that box)."""
    fom_cfg = copy.deepcopy(cfg)
    for s in fom_cfg["subdomains"]:
        s["kind"] = "fom"
    models = schwarz.build_models(fom_cfg)
    ops = {}
    for i, s in enumerate(cfg["subdomains"]):
        if s["kind"] != "rom":
            continue
        m = models[i]
        K = fem.assembled_stiffness(m.box, m.Ke)
        minv = np.repeat(1.0 / m.m, 3)[m.free_dofs, None]
        ops[i] = dict(Phi=np.eye(len(m.free_dofs)), Phi_s=np.eye(len(m.schwarz_dofs)),
                      Kbar=minv * K[np.ix_(m.free_dofs, m.free_dofs)],
                      Bbar=-minv * K[np.ix_(m.free_dofs, m.schwarz_dofs)])
    return ops


def monolithic(cfg, n_steps, E=None):
    """The single-domain FOM on [0, 1] x [0, 0.1]^2 (50 x 5 x 5, rollers at both ends) after n_steps."""
    mono = dict(copy.deepcopy(cfg), subdomains=[I._sub("mono", "fom", (0, 0, 0), (1, 0.1, 0.1), (50, 5, 5),
                                                        (I.ROLLER_X, I.ROLLER_X, 0, 0, 0, 0))], batch=1)
    if E is not None:
        mono["E"] = E
    m = schwarz.build_models(mono)[0]
    u0 = I.initial_displacements(mono, mono["subdomains"][0])
    st, _ = schwarz.run([m], [u0], mono["dt"], n_steps, 1e-10, 50, 2)
    return m, st[0]


def node_map(box, mono_box):
    X, Y = box.coords(), mono_box.coords()
    idx = np.array([np.argmin(np.abs(Y - x).sum(axis=1)) for x in X])
    assert np.abs(Y[idx] - X).max() < 1e-12
    return idx


def rom_fields(model, uh):
    """Full displacement of a full-rank ROM from its reduced state (free DOFs; batch, n_nodes, 3)."""
    out = np.zeros((uh.shape[0], 3 * model.box.n_nodes))
    out[:, model.free_dofs] = uh @ model.Phi.T
    return out.reshape(uh.shape[0], -1, 3)
