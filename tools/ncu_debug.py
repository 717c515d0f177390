"""Where does a 2-rank run stall under ncu?  Prints each step (flushed)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
t0 = time.time()


def say(m):
    print(f"[rank {os.environ.get('RANK')} {time.time() - t0:7.2f}s] {m}", flush=True)


say("start")
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2408_14158_b200 as hfr  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
say("set_device")
torch.zeros(1, device="cuda").sum().item()
say("cuda context")
dist.init_process_group("gloo")
say(f"gloo up: rank {dist.get_rank()} of {dist.get_world_size()}")
comm = hfr.Comm.init(device=local, config=hfr.Config(algo="flat", timeout_ms=120000))
say("comm init")
t = comm.empty(1 << 20, torch.float32)
t.fill_(1.0)
torch.cuda.synchronize()
say("empty + fill")
for i in range(8):
    comm.allreduce(t)
    torch.cuda.synchronize()
    say(f"allreduce {i} status={comm.status()}")
comm.finalize()
say("finalize")
dist.destroy_process_group()
say("done")
