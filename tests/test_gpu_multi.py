"""Multi-process GPU parity (one process per B200, CUDA IPC over NVLink).
Skipped unless >= 2 GPUs are visible (run with `gpurun --gpus 2|4`)."""
import json
import os
import socket

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_multiprocess_parity_protocol_timeout(tmp_path):
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    from paper_2408_14158_b200 import _build
    _build.build()
    import torch.multiprocessing as mp

    from tests import mp_worker
    world = min(torch.cuda.device_count(), 8)
    mp.spawn(mp_worker.entry, args=(world, _free_port(), str(tmp_path), "gpu"), nprocs=world, join=True)
    keep = os.environ.get("HFR_MULTI_OUT")  # copy the per-rank verdicts out (profiles/ evidence)
    for r in range(world):
        res = json.load(open(os.path.join(tmp_path, f"rank{r}.json")))
        if keep:
            os.makedirs(keep, exist_ok=True)
            with open(os.path.join(keep, f"multigpu_n{world}_rank{r}.json"), "w") as f:
                json.dump(res, f, indent=0)
        assert not res["fail"], res["fail"]
        assert "protocol" in res["ok"] and "ddp" in res["ok"] and "1gib" in res["ok"] and "ddp-tail-1" in res["ok"]
        assert "protocol-grid-flat" in res["ok"] and "protocol-grid-auto" in res["ok"]
        assert len(res["ok"]) >= 10
