"""world_size-2 gloo tests on CPU for the host-side N>1 logic."""
import json
import os
import socket

import pytest

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_ipc_exchange_callback_gloo(tmp_path):
    import torch.multiprocessing as mp

    from paper_2408_14158_b200 import _build
    from tests import mp_worker
    _build.build()
    mp.spawn(mp_worker.entry, args=(2, _free_port(), str(tmp_path), "cpu_exchange"), nprocs=2, join=True)
    for r in range(2):
        res = json.load(open(os.path.join(tmp_path, f"rank{r}.json")))
        assert not res["fail"], res["fail"]
        assert res["ok"] == [1, 64, 80, 4096]
