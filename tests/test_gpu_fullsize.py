"""Full-size (BASELINE c3, 41.6M DOFs) parity in the launch configuration bench.py times.

The oracle cannot run c3 end to end in seconds, so it computes sampled outputs one node at a
time: after one controller step from the seeded IC, the final iterate at node p is
    u = u*(p),  a = -f(u*)(p)/m_p,  v = v0 + dt/2 (a0 + a)          (free DOFs)
with u* the predictor (Dirichlet 0, Schwarz s = Pi of the other subdomain's iterate at the
donor nodes).  In c3 every donor node is a free node of its source, whose iterate value is
its own predictor (reading R6), so s is computable from the IC alone.  f and a0 come from
oracle.fem.internal_force_at (element loop over the incident elements of one node).
Properties that hold at any size are checked over several steps: exactly 3 Schwarz
iterations per step (R6) and a finite state.
"""
import numpy as np
import pytest

import osam_inputs as I
from oracle import fem, schwarz, transfer

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_20687_b200 import osam, problem
    osam.lib()
    return problem


class Local:
    """Oracle quantities of one subdomain evaluated node by node from the IC."""

    def __init__(self, sub, faces, cfg):
        self.box = fem.Box(sub["lo"], sub["hi"], sub["nel"])
        self.Ke = fem.hex8_stiffness(self.box.h, cfg["E"], cfg["nu"])
        self.m = fem.lumped_mass(self.box, cfg["rho"])
        self.codes = fem.dof_codes(self.box, sub["dirichlet"], faces.keys())
        self.faces = faces
        u0 = I.initial_displacement(cfg, sub)
        u0[self.codes == fem.DIRICHLET] = 0.0
        self.u0 = u0
        self.dt = cfg["dt"]
        self._a0 = {}

    def a0(self, q):
        q = int(q)
        if q not in self._a0:
            f = fem.internal_force_at(self.box, self.Ke, lambda ids: self.u0[ids], [q])[0]
            self._a0[q] = np.where(self.codes[q] == fem.FREE, -f / self.m[q], 0.0)
        return self._a0[q]

    def predictor(self, q):
        """Iterate value at a free node: u0 + dt v0 + dt^2/2 a0 with v0 = 0."""
        return self.u0[q] + 0.5 * self.dt * self.dt * self.a0(q)


def sample_nodes(box, rng, codes, center):
    X = box.coords()
    d = np.linalg.norm(X - np.asarray(center), axis=1)
    near = np.nonzero(d < 0.15)[0]
    picks = [rng.choice(near, 120, replace=False), rng.choice(box.n_nodes, 40, replace=False)]
    for f in (0, 1):
        fn = box.face_nodes(f)
        picks.append(rng.choice(fn, 30, replace=False))
        inner = fn + (1 if f == 0 else -1)
        picks.append(rng.choice(inner, 20, replace=False))
    corners = [box.node_id(i, j, k) for i in (0, box.nel[0]) for j in (0, box.nel[1]) for k in (0, box.nel[2])]
    picks.append(np.array(corners))
    return np.unique(np.concatenate(picks))


def test_c3_full_size_one_step_sampled(gpu):
    cfg = I.config("c3")
    subs = gpu.build(cfg)
    gpu.set_ics(cfg, subs, device="cuda:0")
    _, iters = gpu.run(cfg, subs, n_steps=1)
    assert iters.tolist() == [[3]]
    boxes = [fem.Box(s["lo"], s["hi"], s["nel"]) for s in cfg["subdomains"]]
    faces = schwarz.detect_schwarz_faces(boxes)
    loc = [Local(s, faces[i], cfg) for i, s in enumerate(cfg["subdomains"])]
    rng = np.random.default_rng(11)
    for i, (sub, L) in enumerate(zip(subs, loc)):
        u, v, a = gpu.fom_state(sub, accel=True)
        nodes = sample_nodes(L.box, rng, L.codes, cfg["ic"]["center"])

        def ustar(q):
            out = np.zeros(3)
            for c in range(3):
                code = L.codes[q, c]
                if code == fem.FREE:
                    out[c] = L.predictor(q)[c]
                elif code == fem.SCHWARZ:
                    ijk = L.box.ijk(q)
                    j = [L.faces[f] for f in sorted(L.faces)
                         if int(ijk[f // 2]) == (L.box.nel[f // 2] if f % 2 else 0)][0]
                    src = loc[j]
                    dn, w = transfer.projector(src.box, L.box.coords(np.array([q])))
                    vals = []
                    for r_ in dn[0]:
                        assert (src.codes[r_] == fem.FREE).all(), "c3 donors are free source nodes"
                        vals.append(src.predictor(r_))
                    out[c] = float(w[0] @ np.array(vals)[:, c])
            return out

        cache = {}

        def value_at(ids):
            res = []
            for q in ids:
                q = int(q)
                if q not in cache:
                    cache[q] = ustar(q)
                res.append(cache[q])
            return np.array(res)

        f = fem.internal_force_at(L.box, L.Ke, value_at, nodes)
        free = L.codes[nodes] == fem.FREE
        ref_u = value_at(nodes)
        ref_a = np.where(free, -f / L.m[nodes, None], 0.0)
        a0 = np.array([L.a0(q) for q in nodes])
        ref_v = np.where(free, 0.5 * L.dt * (a0 + ref_a), 0.0)
        for got, ref, name in ((u[nodes], ref_u, "u"), (v[nodes], ref_v, "v"), (a[nodes], ref_a, "a")):
            err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
            assert err <= 1e-10, (i, name, err)
    # properties at any size over more steps
    _, iters = gpu.run(cfg, subs, n_steps=8)
    assert (iters == 3).all()
    for sub in subs:
        u, v = gpu.fom_state(sub)
        assert np.isfinite(u).all() and np.isfinite(v).all()


def _slab_force(box, Ke, u, i0, i1):
    """Element-loop force of the displacement u (full node-major array) restricted to the x-slab of node
    planes i0..i1 (exact at the slab's interior planes i0+1..i1-1, and at i0 / i1 when they are the
    box's own faces).  Returns f on planes i0..i1 as (nz+1, ny+1, i1-i0+1, 3)."""
    nn = box.nn
    sub = fem.Box((box.lo[0] + i0 * box.h[0], box.lo[1], box.lo[2]),
                  (box.lo[0] + i1 * box.h[0], box.hi[1], box.hi[2]), (i1 - i0, box.nel[1], box.nel[2]))
    us = u.reshape(nn[2], nn[1], nn[0], 3)[:, :, i0:i1 + 1].reshape(-1, 3)
    return fem.internal_force(sub, Ke, us).reshape(nn[2], nn[1], i1 - i0 + 1, 3)


def test_c4_full_size_one_step_sampled(gpu):
    """BASELINE c4 at full size (256^3 FOM between two r = 200 ROMs on 80^3 meshes), one controller step,
    with the seeded stand-in operators bench.py uses.  The oracle rebuilds the final iterate: the ROMs in
    full (their Schwarz data are the FOM's predictor at donor nodes, R6), the FOM on x-slabs (its Schwarz
    data are the lifted ROM predictors).  Compared: u^, v^, a^ of both ROMs; u, v, a of the FOM on every
    node of five slabs (both Schwarz faces, both ROM donor regions, the pulse centre)."""
    cfg = I.config("c4")
    ops = gpu.synthetic_rom_ops(cfg)
    subs = gpu.build(cfg, ops)
    gpu.set_ics(cfg, subs, device="cuda:0")
    _, iters = gpu.run(cfg, subs, n_steps=1)
    assert 2 <= int(iters[0, 0]) <= 3
    models = schwarz.build_models(cfg, rom_ops=ops)
    L, Cm, R = models
    dt = cfg["dt"]
    u0s = [I.initial_displacements(cfg, s) for s in cfg["subdomains"]]
    box = Cm.box
    free = Cm.codes == fem.FREE
    uC0 = np.array(u0s[1][0])
    uC0[Cm.codes == fem.DIRICHLET] = 0.0
    m = Cm.m.reshape(box.nn[2], box.nn[1], box.nn[0])
    freeg = free.reshape(box.nn[2], box.nn[1], box.nn[0], 3)

    def a0_planes(i0, i1):  # a0 on planes i0+1..i1-1 (or including box faces)
        f = _slab_force(box, Cm.Ke, uC0, i0, i1)
        a = -f / m[:, :, i0:i1 + 1, None]
        return np.where(freeg[:, :, i0:i1 + 1], a, 0.0)

    # FOM iterate displacement u* at free nodes = predictor (v0 = 0), filled where the ROMs read it
    u_it = uC0.reshape(box.nn[2], box.nn[1], box.nn[0], 3).copy()
    for (i0, i1) in ((23, 28), (227, 232)):
        a = a0_planes(i0, i1)
        u_it[:, :, i0 + 1:i1] = np.where(freeg[:, :, i0 + 1:i1], u_it[:, :, i0 + 1:i1] + 0.5 * dt * dt * a[:, :, 1:-1],
                                         u_it[:, :, i0 + 1:i1])
    stC = dict(u=u_it.reshape(1, -1, 3))
    # ROMs: s from the FOM iterate, then one OpInf step from the IC
    rom_ref = {}
    for k, mdl in ((0, L), (2, R)):
        st0 = mdl.init_state(u0s[k])
        s = mdl.gather_s([None, [stC, stC], None], models)   # single-substep traces
        rom_ref[k] = mdl.advance(st0, s)
    for k in (0, 2):
        uh, vh, ah = gpu.rom_state(subs[k], accel=True)
        for got, ref in ((uh, rom_ref[k]["uh"]), (vh, rom_ref[k]["vh"]), (ah, rom_ref[k]["ah"])):
            assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref), k
    # FOM: Schwarz values = lifted ROM predictors; slabs checked on every node of their interior planes
    sC = Cm.gather_s([[rom_ref[0]] * 2, None, [rom_ref[2]] * 2], models)[0]
    ustar_all = u_it.reshape(-1, 3).copy()
    ustar_all.reshape(-1)[Cm.schwarz_dofs] = sC
    u, v, a = gpu.fom_state(subs[1], accel=True)
    for (i0, i1) in ((0, 5), (21, 30), (123, 133), (225, 234), (251, 256)):
        a0 = a0_planes(max(i0 - 1, 0), min(i1 + 1, box.nel[0]))
        lo = 1 if i0 > 0 else 0
        us = ustar_all.reshape(box.nn[2], box.nn[1], box.nn[0], 3).copy()
        pl = slice(i0, i1 + 1)
        a0s = a0[:, :, lo:lo + (i1 - i0 + 1)]
        us[:, :, pl] = np.where(freeg[:, :, pl], uC0.reshape(us.shape)[:, :, pl] + 0.5 * dt * dt * a0s, us[:, :, pl])
        f = _slab_force(box, Cm.Ke, us.reshape(-1, 3), i0, i1)
        ref_a = np.where(freeg[:, :, pl], -f / m[:, :, pl, None], 0.0)
        ref_v = np.where(freeg[:, :, pl], 0.5 * dt * (a0s + ref_a), 0.0)
        ref_u = us[:, :, pl]
        j0, j1 = (i0 + 1 if i0 > 0 else 0), (i1 - 1 if i1 < box.nel[0] else i1)  # exact planes of the slab
        sel = slice(j0 - i0, j1 - i0 + 1)
        for got, ref, name in ((u, ref_u, "u"), (v, ref_v, "v"), (a, ref_a, "a")):
            g = got.reshape(box.nn[2], box.nn[1], box.nn[0], 3)[:, :, j0:j1 + 1]
            r = ref[:, :, sel]
            assert np.linalg.norm(g - r) <= 1e-10 * max(np.linalg.norm(r), 1e-300), (i0, name)
