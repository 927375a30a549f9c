"""End-to-end pins of the oracle's FOM-ROM and ROM-ROM coupling: with full-rank intrusive
operators (tests/fullrank.py) a conformal coupled run equals the monolithic FOM on the union of the boxes."""
import numpy as np
import pytest

import fullrank as F
import osam_inputs as I
from oracle import fem, schwarz


def _coupled(cfg, n_steps, ops, e=None):
    models = schwarz.build_models(cfg, ops, e)
    u0s = [I.initial_displacements(cfg, s) for s in cfg["subdomains"]]
    states, iters = schwarz.run(models, u0s, cfg["dt"], n_steps, cfg["tol"], 50, 2)
    return models, states, iters


@pytest.mark.parametrize("kinds", [("fom", "rom"), ("rom", "fom"), ("rom", "rom")])
def test_full_rank_rom_coupling_equals_monolithic(kinds):
    cfg = F.conformal_cfg(kinds)
    n = 60
    models, states, iters = _coupled(cfg, n, F.full_rank_ops(cfg))
    mm, ms = F.monolithic(cfg, n)
    for m, st in zip(models, states):
        idx = F.node_map(m.box, mm.box)
        u = st["u"][0] if m.kind == "fom" else F.rom_fields(m, st["uh"])[0]
        free = m.codes == fem.FREE
        ref = ms["u"][0][idx]
        assert np.linalg.norm(np.where(free, u - ref, 0)) <= 1e-12 * np.linalg.norm(ref), kinds
    assert (iters == 3).all()


def test_full_rank_batched_rom_rom_equals_monolithic_per_sample():
    """Batched ROM-ROM with per-sample moduli: sample b equals the monolithic FOM at E_b = e_b E."""
    e = [0.8, 1.0, 1.2]
    cfg = F.conformal_cfg(("rom", "rom"), batch=e)
    n = 40
    models, states, iters = _coupled(cfg, n, F.full_rank_ops(cfg), np.array(e))
    for b, eb in enumerate(e):
        mm, ms = F.monolithic(cfg, n, E=I.E0 * eb)
        for m, st in zip(models, states):
            idx = F.node_map(m.box, mm.box)
            u = F.rom_fields(m, st["uh"])[b]
            free = m.codes == fem.FREE
            ref = ms["u"][0][idx]
            assert np.linalg.norm(np.where(free, u - ref, 0)) <= 1e-12 * np.linalg.norm(ref), (b, m.spec["name"])
