"""Config #5 machinery (tests/long_run.py) at a reduced size: invariants series,
LBFIELD checkpoints and oracle checkpoint-restart parity <= 1e-12."""
import os
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("gravity", [0.0, 1e-4])
def test_long_run_small(gravity):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import long_run
    res = long_run.main(["--lx", "256", "--ly", "512", "--steps", "600", "--every", "50",
                         "--ckpt-every", "200", "--check", "5", "--gravity", str(gravity)])
    assert len(res["checkpoint_restart_parity"]) == 3
    assert res["max_checkpoint_err"] < 1e-12
    assert abs(res["rel_mass_drift"]) < 1e-12
    assert res["min_rho_final"] > 0.5


def test_long_run_config5_n8_geometry_reduced():
    """BASELINE configs[4] at its N = 8 geometry — 2048x4096 as 8 X-slabs of 256
    columns, an in-process peer ring on one GPU (two-step kernel + staged
    pull) — for 600 of the 10^4 steps: the library restarts from every LBFIELD
    checkpoint (file -> set_state), each checkpoint is bitwise equal to an
    unsplit lattice stepped from memory (N == 1), and the oracle restarted from
    it agrees within 1e-12 after 4 steps."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import long_run
    res = long_run.main(["--lx", "2048", "--ly", "4096", "--nslabs", "8", "--compare-n1", "--steps", "600",
                         "--every", "100", "--ckpt-every", "200", "--check", "4"])
    assert len(res["checkpoint_restart_parity"]) == 3
    assert res["max_checkpoint_err"] < 1e-12
    assert len(res["unsplit_bitwise"]) == 4 and res["all_bitwise_equal_to_unsplit"]
    assert abs(res["rel_mass_drift"]) < 1e-12
    assert all(abs(r["unsplit_mass_rel_diff"]) < 1e-13 for r in res["series"])
    assert res["min_rho_final"] > 0.5
