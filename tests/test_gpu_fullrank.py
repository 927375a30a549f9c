"""GPU end-to-end pins of the FOM-ROM / ROM-ROM coupling paths: with full-rank intrusive operators
(tests/fullrank.py) libosam.so's conformal coupled runs must equal the monolithic FOM on the union (computed by
the oracle), per sample for batched ROMs (tensor-core and CUDA-core ROM paths)."""
import numpy as np
import pytest

import fullrank as F
import osam_inputs as I
from oracle import fem, schwarz

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_20687_b200 import osam, problem
    osam.lib()
    return problem


def _gpu_fields(problem, cfg, subs, models):
    out = []
    for sub, m in zip(subs, models):
        if m.kind == "fom":
            out.append(problem.fom_state(sub)[0][None])
        else:
            out.append(F.rom_fields(m, problem.rom_state(sub)[0]))
    return out


@pytest.mark.parametrize("kinds", [("fom", "rom"), ("rom", "fom"), ("rom", "rom")])
def test_gpu_full_rank_rom_coupling_equals_monolithic(gpu, kinds):
    cfg = F.conformal_cfg(kinds)
    ops = F.full_rank_ops(cfg)
    n = 60
    subs = gpu.build(cfg, ops)
    gpu.set_ics(cfg, subs, device="cuda:0")
    _, iters = gpu.run(cfg, subs, n_steps=n)
    assert (iters == 3).all()
    models = schwarz.build_models(cfg, ops)
    mm, ms = F.monolithic(cfg, n)
    for u, m in zip(_gpu_fields(gpu, cfg, subs, models), models):
        idx = F.node_map(m.box, mm.box)
        free = m.codes == fem.FREE
        ref = ms["u"][0][idx]
        assert np.linalg.norm(np.where(free, u[0] - ref, 0)) <= TOL * np.linalg.norm(ref), kinds


@pytest.mark.parametrize("tc", ["1", "0"])
def test_gpu_full_rank_batched_rom_rom_equals_monolithic_per_sample(gpu, monkeypatch, tc):
    monkeypatch.setenv("OSAM_ROM_TC", tc)
    e = [0.8, 1.0, 1.2]
    cfg = F.conformal_cfg(("rom", "rom"), batch=e)
    ops = F.full_rank_ops(cfg)
    n = 40
    subs = gpu.build(cfg, ops)
    gpu.set_ics(cfg, subs, device="cuda:0")
    gpu.run(cfg, subs, n_steps=n)
    models = schwarz.build_models(cfg, ops, np.array(e))
    fields = _gpu_fields(gpu, cfg, subs, models)
    for b, eb in enumerate(e):
        mm, ms = F.monolithic(cfg, n, E=I.E0 * eb)
        for u, m in zip(fields, models):
            idx = F.node_map(m.box, mm.box)
            free = m.codes == fem.FREE
            ref = ms["u"][0][idx]
            assert np.linalg.norm(np.where(free, u[b] - ref, 0)) <= TOL * np.linalg.norm(ref), (b, tc)
