"""The tile shapes of the tiled K1 (kernels_fom.cu k1_shape: k1a 32 x 4, a warp per x-row; k1b 16 x 8, a
warp per two 16-node rows, picked for x-ragged boxes such as c3's; k1c 48 x 2, three warps over two rows) on the tiled-K1 parity cases of
tests/test_gpu_parity.py, each forced with OSAM_K1_SHAPE: against the oracle, and bitwise between the
controllers."""
import pytest

from test_gpu_parity import (  # noqa: F401  (re-collected here under both shapes)
    gpu, test_bitwise_repeatable, test_c1_substeps_xi, test_graph_controller_equals_host_loop_bitwise,
    test_max_iters_reached_keeps_last_iterate, test_scaled_c3_several_tiles_ragged,
    test_scaled_c4_fom_between_two_roms, test_single_fom_degenerate_and_ragged,
    test_xlast_column_excluded_c1_variant, test_xlast_column_excluded_c4_topology)

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["k1a", "k1b", "k1c"])
def k1_shape(monkeypatch, request):
    monkeypatch.setenv("OSAM_GATHER_MAX", "0")          # the tiled K1 at every size
    monkeypatch.setenv("OSAM_K1_SHAPE", {"k1a": "0", "k1b": "1", "k1c": "2"}[request.param])


@pytest.mark.timeout(300, method="thread")
@pytest.mark.parametrize("created,stepped", [("1", "0"), ("0", "1"), ("2", "1")])
def test_tmaps_follow_the_shape_at_bind(gpu, monkeypatch, created, stepped):
    """The TMA boxes follow the tile shape, which is fixed only at bind (it depends on the Schwarz faces):
    subdomains created (and given their IC) under one shape and stepped under the other still match the
    oracle, because bind encodes the descriptors again.  Without that re-encoding the kernel waits for TMA
    bytes that never arrive (checked once with such a build: it hangs), hence the timeout."""
    from test_gpu_parity import compare, oracle_run
    import osam_inputs as I
    cfg = I.scaled(I.config("c3"), 8.0)
    monkeypatch.setenv("OSAM_K1_SHAPE", created)
    subs = gpu.build(cfg)
    gpu.set_ics(cfg, subs, device="cuda:0")
    monkeypatch.setenv("OSAM_K1_SHAPE", stepped)
    n = 6
    _, iters = gpu.run(cfg, subs, n_steps=n)
    models, states, it_ref, _ = oracle_run(cfg, n, e=gpu.e_scale(cfg))
    assert (iters.reshape(-1) == it_ref.reshape(-1)).all()
    compare(gpu, subs, models, states)
