"""CPU tests of the HaiScale-DDP bucket planner (§8 a6)."""
import pytest

from paper_2408_14158_b200.ddp import plan_buckets


def test_plan_tiles_exactly():
    numels = [10, 0, 7, 33, 1, 64]
    ranges, buckets, members = plan_buckets(numels, 16)
    assert ranges[0] == (0, 10) and ranges[-1] == (51, 115)
    assert buckets[0] == (0, 16) and buckets[-1] == (112, 115)
    covered = []
    for s, e in buckets:
        covered.extend(range(s, e))
    assert covered == list(range(115))
    # every member overlaps its bucket; every overlapping param is a member
    for k, (s, e) in enumerate(buckets):
        want = [i for i, (a, b) in enumerate(ranges) if b > a and a < e and b > s]
        assert members[k] == want


@pytest.mark.parametrize("bucket", [1, 3, 64, 1000])
def test_ready_order_launches_each_bucket_once(bucket):
    numels = [5, 17, 3, 100, 2, 40]
    _, buckets, members = plan_buckets(numels, bucket)
    pending = [len(m) for m in members]
    launched = []
    for i in range(len(numels)):
        for k, mem in enumerate(members):
            if i in mem:
                pending[k] -= 1
                if pending[k] == 0:
                    launched.append(k)
    assert sorted(launched) == list(range(len(buckets)))
    assert launched == sorted(launched)  # backward order fills buckets in order


def test_c5_bucket_count():
    """config 5: 7.0e9 bf16 = 14.0e9 B -> 208 x 64 MiB + one 41,356,288 B bucket."""
    import tools.ddp_overlap as d
    numels = [o * i for _, o, i in d.llama7b_layout()]
    assert sum(numels) == 7_000_000_000
    _, buckets, _ = plan_buckets(numels, (64 << 20) // 2)
    assert len(buckets) == 209
    assert (buckets[-1][1] - buckets[-1][0]) * 2 == 41_356_288


def test_bad_bucket():
    with pytest.raises(ValueError):
        plan_buckets([1], 0)


class _FakeComm:
    """Records (config, bucket offset) per allreduce; CPU tensors only."""

    def __init__(self, scale=1.0):
        from paper_2408_14158_b200 import Config
        self.config = Config(scale=scale)
        self.calls = []

    def empty(self, numel, dtype):
        import torch
        return torch.zeros(numel, dtype=dtype)

    def set_config(self, cfg):
        self.config = cfg

    def allreduce(self, t, async_op=False, stream=None):
        self.calls.append((self.config, t.data_ptr()))

        class _W:
            def wait(self, stream=None):
                pass
        return _W()


@pytest.mark.parametrize("tail_from", [None, 2, 4])
def test_tail_config_covers_exactly_the_late_buckets(tail_from):
    import torch
    from paper_2408_14158_b200.ddp import HaiScaleDDP
    numels = [40, 17, 100, 3, 60]
    comm = _FakeComm(scale=0.25)
    overlap = HaiScaleDDP.derive(comm, max_ctas=8)
    tail = HaiScaleDDP.derive(comm, max_ctas=0, algo="flat")
    ddp = HaiScaleDDP(comm, numels, torch.float32, bucket_bytes=16 * 4, config=overlap, tail_config=tail,
                      tail_from=tail_from)
    base = comm.config
    tf = len(numels) - 1 if tail_from is None else tail_from
    for step in range(2):
        comm.calls = []
        for i in range(len(numels)):
            ddp.mark_ready(i)
        ddp.finish()
        assert comm.config is base, "finish() restores the comm's config"
        assert len(comm.calls) == len(ddp.bucket_ranges)
        esz = 4
        for cfg, ptr in comm.calls:
            k = (ptr - ddp.arena.data_ptr()) // esz // ddp.bucket_elems
            last_member = max(ddp.bucket_params[k])
            assert cfg is (tail if last_member >= tf else overlap), (k, cfg)
            assert cfg.scale == 0.25
    assert ddp.stats.tail == 2 * sum(1 for m in ddp.bucket_params if max(m) >= tf)


def test_no_configs_leaves_comm_config_alone():
    import torch
    from paper_2408_14158_b200.ddp import HaiScaleDDP
    comm = _FakeComm()
    base = comm.config
    ddp = HaiScaleDDP(comm, [10, 20], torch.float32, bucket_bytes=32)
    for i in range(2):
        ddp.mark_ready(i)
    ddp.finish()
    assert all(c is base for c, _ in comm.calls) and ddp.stats.tail == 0


def test_c5_tail_buckets_are_the_embedding_gemm_buckets():
    """C5 tail (tools/ddp_overlap.py --tail 1): the buckets completed by the
    last gradient GEMM (embedding) or later — 9 of the 209, the last one ragged."""
    import tools.ddp_overlap as d
    params = d.llama7b_layout()
    numels = [o * i for _, o, i in params]
    tail_from = [nm for nm, _, _ in params].index("embed")
    _, buckets, members = plan_buckets(numels, (64 << 20) // 2)
    tail = [k for k, m in enumerate(members) if max(m) >= tail_from]
    assert tail == list(range(200, 209))
    assert 7 * (64 << 20) // 2 < params[tail_from][1] * params[tail_from][2] < 8 * (64 << 20) // 2  # 7.8 buckets over 9


def test_config_scale_must_match_the_comm():
    """a DDP config built from scratch (scale 1.0) on a comm that
    averages (scale 1/n) would silently sum — refused."""
    import torch
    from paper_2408_14158_b200 import Config
    from paper_2408_14158_b200.ddp import HaiScaleDDP
    comm = _FakeComm(scale=0.125)
    with pytest.raises(ValueError):
        HaiScaleDDP(comm, [10, 20], torch.float32, bucket_bytes=32, config=Config(max_ctas=32))
    with pytest.raises(ValueError):
        HaiScaleDDP(comm, [10, 20], torch.float32, bucket_bytes=32, tail_config=Config())
    ddp = HaiScaleDDP(comm, [10, 20], torch.float32, bucket_bytes=32, tail_config=HaiScaleDDP.derive(comm))
    assert ddp.tail_config.scale == 0.125
