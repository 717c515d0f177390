import sys, numpy as np, torch
sys.path.insert(0, '.')
import hfr_inputs as gen
import paper_2408_14158_b200 as hfr
from oracle import hfr_oracle as O
from tests.gpu_util import to_torch, to_numpy
for n in (3, 4):
  for dist in ("normal", "int"):
    comm = hfr.Comm.virtual_ranks(n, 0, hfr.Config(timeout_ms=5000, algo="dbt", chunk_elems=512))
    N = 4096
    xs = gen.rank_inputs(n, N, gen.FP16, dist, seed_base=1000 + N)
    bufs = comm.empty(N, torch.float16)
    for b, x in zip(bufs, xs): b.copy_(to_torch(x, "cuda:0"))
    comm.allreduce_virtual(bufs); torch.cuda.synchronize()
    want = O.allreduce(xs, "dbt", chunk_elems=512)[0]
    for r, b in enumerate(bufs):
        g = to_numpy(b)
        bad = np.flatnonzero(g.view(np.uint16) != want.view(np.uint16))
        chunks = sorted(set((bad // 512).tolist()))
        print(n, dist, "rank", r, "bad", bad.size, "chunks", chunks, "first", bad[:4].tolist(), g[bad[:4]].tolist(), want[bad[:4]].tolist())
    comm.finalize()
