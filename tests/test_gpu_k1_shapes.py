"""Both tile shapes of the tiled K1 (kernels_fom.cu k1_shape: k1a 32 x 4, a warp per x-row; k1b 16 x 8, a
warp per two 16-node rows, picked for x-ragged boxes such as c3's) on the tiled-K1 parity cases of
tests/test_gpu_parity.py, each forced with OSAM_K1_SHAPE: against the oracle, and bitwise between the
controllers."""
import pytest

from test_gpu_parity import (  # noqa: F401  (re-collected here under both shapes)
    gpu, test_bitwise_repeatable, test_c1_substeps_xi, test_graph_controller_equals_host_loop_bitwise,
    test_max_iters_reached_keeps_last_iterate, test_scaled_c3_several_tiles_ragged,
    test_scaled_c4_fom_between_two_roms, test_single_fom_degenerate_and_ragged,
    test_xlast_column_excluded_c1_variant, test_xlast_column_excluded_c4_topology)

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["k1a", "k1b"])
def k1_shape(monkeypatch, request):
    monkeypatch.setenv("OSAM_GATHER_MAX", "0")          # the tiled K1 at every size
    monkeypatch.setenv("OSAM_K1_SHAPE", "0" if request.param == "k1a" else "1")
