"""Multi-GPU tests (need >= 2 visible GPUs; skipped otherwise)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs 2 GPUs")
def test_domain_partitioned_operator_nccl(tmp_path):
    out = tmp_path / "dist.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533",
           str(Path(__file__).with_name("dist_gpu_check.py")), str(out)]
    subprocess.run(cmd, check=True, timeout=900)
    rep = json.loads(out.read_text())
    assert rep.pop("volume_reports_equal")     # partitioned == emulation byte accounting
    for prec in ("single", "mixed"):
        assert rep.pop(f"{prec}_streamed_equal")["equal"], prec
        assert rep.pop(f"{prec}_fused_equal")["equal"], prec      # fused == NCCL p2p
    for key, r in rep.items():
        # reference staging + direct-plan reduction order: the NCCL exchange
        # reproduces the one-process emulation; only the cross-rank f64 dot
        # sums differ (alpha/beta are cast to f32)
        if key.endswith("reference"):
            assert r["vs_emulation"] <= 1e-6, (key, r)
            assert r["vs_oracle"] <= 1e-6, (key, r)       # the reference's P_d run
        # P_d > 1 itself changes the rounding (per-rank fp16 partials in
        # mixed mode): the reference moves by 5e-5 (single) / 2.4e-2 (mixed)
        # between P_d = 2 and P_d = 1 on this problem (oracle)
        assert r["vs_single_gpu"] <= (5e-4 if key.startswith("single") else 5e-2), (key, r)
