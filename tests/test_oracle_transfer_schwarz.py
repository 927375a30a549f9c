"""Pins for oracle/transfer.py and oracle/schwarz.py."""
import json
import os

import numpy as np
import pytest

import osam_inputs as I
from oracle import fem, schwarz, transfer

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_transfer_reproduces_trilinear_fields():
    box = fem.Box((0.45, 0, 0), (1, 1, 1), (11, 7, 9))
    rng = np.random.default_rng(0)
    X = box.lo + rng.random((200, 3)) * (box.hi - box.lo)
    c = rng.standard_normal((8, 3))
    def field(P):      # span{1, x, y, z, xy, yz, zx, xyz} per component
        x, y, z = P[..., 0], P[..., 1], P[..., 2]
        basis = np.stack([np.ones_like(x), x, y, z, x * y, y * z, z * x, x * y * z], axis=-1)
        return basis @ c
    Y = box.coords()
    nodes, w = transfer.projector(box, X)
    s = transfer.apply(nodes, w, lambda ids: field(Y)[ids][None])[0]
    assert np.abs(s - field(X)).max() <= 1e-13 * np.abs(field(X)).max()
    assert np.allclose(w.sum(axis=1), 1.0, rtol=0, atol=1e-15)
    assert (w >= -1e-15).all()


def test_transfer_coincident_nodes_select():
    box = fem.Box((0, 0, 0), (0.6, 0.1, 0.1), (30, 5, 5))
    Y = box.coords()
    ids = np.array([0, 17, 300, box.n_nodes - 1])
    nodes, w = transfer.projector(box, Y[ids])
    vals = np.random.default_rng(1).standard_normal((box.n_nodes, 3))
    s = transfer.apply(nodes, w, lambda q: vals[q][None])[0]
    assert np.array_equal(s, vals[ids])


def test_transfer_outside_raises():
    box = fem.Box((0.4, 0, 0), (1, 0.1, 0.1), (24, 4, 4))
    with pytest.raises(transfer.OverlapError):
        transfer.projector(box, np.array([[0.39, 0.05, 0.05]]))
    transfer.projector(box, np.array([[0.4 - 1e-12, 0.05, 0.05]]))   # within tolerance


@pytest.mark.parametrize("name,expected", [
    ("c1", [{1: 1}, {0: 0}]),
    ("c3", [{1: 1}, {0: 0}]),
    ("c4", [{1: 1}, {0: 0, 1: 2}, {0: 1}]),
    ("c5", [{1: 1}, {0: 0}]),
])
def test_detect_schwarz_faces(name, expected):
    cfg = I.config(name)
    boxes = [fem.Box(s["lo"], s["hi"], s["nel"]) for s in cfg["subdomains"]]
    assert schwarz.detect_schwarz_faces(boxes) == expected


def test_dof_counts_c1_c2():
    cfg = I.config("c1")
    ms = schwarz.build_models(cfg)
    # omega1: 31x6x6 = 1116 nodes; Schwarz face x=0.6: 36 nodes x 3; roller x=0: 36 x-components
    assert ms[0].box.n_nodes == 1116 and len(ms[0].schwarz_dofs) == 108
    assert len(ms[0].free_dofs) == 3 * 1116 - 108 - 36
    assert ms[1].box.n_nodes == 625 and len(ms[1].schwarz_dofs) == 75
    g = json.load(open(os.path.join(GOLD, "survey_crosscheck.json")))["c2"]["offline"]
    c2 = I.config("c2")
    boxes = [fem.Box(s["lo"], s["hi"], s["nel"]) for s in c2["subdomains"]]
    faces = schwarz.detect_schwarz_faces(boxes)
    codes = fem.dof_codes(boxes[1], c2["subdomains"][1]["dirichlet"], faces[1].keys())
    assert int((codes == fem.FREE).sum()) == g["N_free"] == 3 * 7381 - 363 - 121


def _run(cfg, n_steps=None, trace=False):
    models = schwarz.build_models(cfg)
    u0s = [I.initial_displacements(cfg, s) for s in cfg["subdomains"]]
    states = [m.init_state(u0) for m, u0 in zip(models, u0s)]
    iters, traces = [], []
    for _ in range(n_steps or cfg["n_steps"]):
        tr = []
        states, it = schwarz.controller_step(models, states, cfg["tol"], trace=tr)
        iters.append(it)
        traces.append(tr)
    return models, states, np.array(iters), traces


def test_c1_matches_independent_prototype_and_three_iterations():
    g = json.load(open(os.path.join(GOLD, "survey_crosscheck.json")))["c1"]
    cfg = I.config("c1")
    models = schwarz.build_models(cfg)
    u0s = [I.initial_displacements(cfg, s) for s in cfg["subdomains"]]
    states = [m.init_state(u0) for m, u0 in zip(models, u0s)]
    got = {}
    for k in range(cfg["n_steps"]):
        tr = []
        states, it = schwarz.controller_step(models, states, cfg["tol"], trace=tr)
        # R6: every step takes exactly 3 iterations and the 3rd iteration changes nothing
        assert it.tolist() == [3]
        assert tr[-1][1][0] == 0.0 and tr[0][1][0] > 0.0
        if k in (0, 199):
            got[k] = [[np.linalg.norm(s["u"]), np.linalg.norm(s["v"]), s["u"][0, :, 0].max()] for s in states]
    for k, key in ((0, "after_step_1"), (199, "after_step_200")):
        for i, name in enumerate(("omega1", "omega2")):
            assert np.allclose(got[k][i], g[key][name], rtol=g["rel_tol"], atol=0)


def test_conformal_fom_fom_equals_monolithic():
    """Conformal FOM-FOM O-SAM = single-domain FOM on the union (SURVEY finding 2)."""
    cfg = I.config("c1")
    cfg["subdomains"][1] = dict(cfg["subdomains"][1], nel=(30, 5, 5))
    cfg["dt"] = 0.5 * 0.02 / fem.p_wave_speed(1e9, 0.25, 1000.0)
    n = 200
    models, states, iters, _ = _run(cfg, n)
    mono_cfg = dict(cfg, subdomains=[I._sub("mono", "fom", (0, 0, 0), (1, 0.1, 0.1), (50, 5, 5),
                                             (I.ROLLER_X, I.ROLLER_X, 0, 0, 0, 0))])
    mm, ms, _, _ = _run(mono_cfg, n)
    Ym = mm[0].box.coords()
    for m, st in zip(models, states):
        X = m.box.coords()
        idx = np.array([np.argmin(np.abs(Ym - x).sum(axis=1)) for x in X])
        assert np.abs(Ym[idx] - X).max() < 1e-12
        ref_u = ms[0]["u"][0][idx]
        assert np.linalg.norm(st["u"][0] - ref_u) <= 1e-12 * np.linalg.norm(ref_u)
        free = m.codes == fem.FREE
        ref_v = ms[0]["v"][0][idx]
        assert np.linalg.norm((st["v"][0] - ref_v)[free]) <= 1e-12 * np.linalg.norm(ref_v[free])
