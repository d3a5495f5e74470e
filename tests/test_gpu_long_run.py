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
