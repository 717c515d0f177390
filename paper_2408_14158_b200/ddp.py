"""HaiScale-style DDP gradient bucketing over HFReduce (§8 row a6).

PAPER.md:449-453 (§5 "HaiScale DDP Overlap AllReduce in Training"): "During the
backpropagation phase, HaiScale DDP performs an asynchronous allreduce
operation on the computed gradients, allowing this communication to overlap
with the computation involved in backpropagation."

B200 recast: every gradient lives in ONE symmetric peer-mapped arena
(hfr_mem_alloc) laid out in backward order, cut into fixed-size buckets
(64 MiB by default, config 5).  As the backward pass finishes the last
gradient touching a bucket, the bucket's hfr_allreduce is enqueued
asynchronously: the comm side stream waits on an event recorded on the
compute stream, so the reduction overlaps the rest of the backward.  finish()
orders every bucket's completion back onto the compute stream before the
optimizer step.  The comm kernels are capped at `max_ctas` CTAs so they leave
most SMs to the backward GEMMs (unlike the paper's copy-engine HFReduce,
PAPER.md:375, an SM-driven allreduce is not free — DESIGN.md §6).

Measured on 4 B200s with a 7e9-parameter LLaMA-shaped backward (C5, median
of 15 interleaved repetitions): the best bit-exact setting is FLAT with
Config(max_ctas=32..40, threads=128, stream_gate=1, flat_staging=1) — small
register-staged comm CTAs (no shared memory) share SMs with the GEMM CTAs —
plus a full-width tail_config for the buckets completed by the last gradient
GEMM, for an overlap of 0.90-0.95 over runs (0.91 without the tail); algo "nvls"
(order-relaxed) with 16 CTAs reaches 0.98-0.99.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple


def plan_buckets(numels: Sequence[int], bucket_elems: int) -> Tuple[List[Tuple[int, int]], List[Tuple[int, int]],
                                                                    List[List[int]]]:
    """Lay parameters out back to back in the given (backward) order and cut
    the arena into buckets of `bucket_elems` elements (the last one ragged).

    Returns (param_ranges, bucket_ranges, bucket_params) where param_ranges[i]
    = [start, end) of parameter i in the arena, bucket_ranges[k] = [start, end)
    of bucket k, and bucket_params[k] = indices of the parameters overlapping
    bucket k (a bucket is ready once all of them are written)."""
    if bucket_elems <= 0:
        raise ValueError("bucket_elems must be positive")
    ranges = []
    off = 0
    for m in numels:
        if m < 0:
            raise ValueError("negative numel")
        ranges.append((off, off + m))
        off += m
    total = off
    buckets = [(s, min(s + bucket_elems, total)) for s in range(0, total, bucket_elems)]
    members: List[List[int]] = [[] for _ in buckets]
    for i, (s, e) in enumerate(ranges):
        if e == s:
            continue
        for k in range(s // bucket_elems, (e - 1) // bucket_elems + 1):
            members[k].append(i)
    return ranges, buckets, members


@dataclass
class BucketStats:
    launched: int = 0
    bytes: int = 0
    tail: int = 0   # buckets launched with tail_config


class HaiScaleDDP:
    """Gradient arena + asynchronous bucketed allreduce for one rank.

    Usage per step:
        ddp.zero_grad()                     (optional; the backward may overwrite instead)
        for i in backward order: write ddp.grad(i); ddp.mark_ready(i, stream)
        ddp.finish(stream)                  (stream waits for every bucket)
    """

    def __init__(self, comm, numels: Sequence[int], dtype, bucket_bytes: int = 64 << 20,
                 config=None, tail_config=None, tail_from: Optional[int] = None):
        """`config`: the comm config for buckets that overlap the backward
        (e.g. few small CTAs); `tail_config`: the config for the buckets
        completed by marking parameter `tail_from` (backward order) or a later
        one — the last gradient GEMM of the step; nothing is left to overlap
        them with, so they may take the whole GPU.  tail_from None: the last
        parameter.  tail_config None: `config` throughout; both None: the
        comm's current config; tail_config without config: ValueError.
        Every rank makes the same choice for the same bucket (collective
        contract, include/hfr.h)."""
        import torch
        if tail_config is not None and config is None:
            raise ValueError("tail_config needs config (the comm's config is not restored otherwise)")
        self.comm = comm
        self.config = config
        self.tail_config = tail_config
        self.tail_from = len(numels) - 1 if tail_from is None else tail_from
        self.dtype = dtype
        esz = torch.tensor([], dtype=dtype).element_size()
        self.bucket_elems = max(1, bucket_bytes // esz)
        self.param_ranges, self.bucket_ranges, self.bucket_params = plan_buckets(list(numels), self.bucket_elems)
        self.total = self.param_ranges[-1][1] if self.param_ranges else 0
        self.arena = comm.empty(max(1, self.total), dtype)
        if isinstance(self.arena, list):
            raise ValueError("HaiScaleDDP needs a real (one rank per process) comm")
        self._pending = [len(m) for m in self.bucket_params]
        self._active = None
        self._bucket_of_param: List[List[int]] = [[] for _ in numels]
        for k, mem in enumerate(self.bucket_params):
            for i in mem:
                self._bucket_of_param[i].append(k)
        self._works = []
        self.stats = BucketStats()

    def zero_grad(self):
        self.arena.zero_()

    def grad(self, i: int):
        s, e = self.param_ranges[i]
        return self.arena[s:e]

    def bucket(self, k: int):
        s, e = self.bucket_ranges[k]
        return self.arena[s:e]

    def reset(self):
        self._pending = [len(m) for m in self.bucket_params]
        self._works = []
        self._active = None  # re-apply the configs each step (the caller may have changed the comm's)

    def _use(self, cfg):
        if cfg is not None and cfg is not self._active:
            self.comm.set_config(cfg)
            self._active = cfg

    def mark_ready(self, i: int, stream=None):
        """Parameter i's gradient has been enqueued on `stream`; launch the
        allreduce of every bucket that just became complete.  Buckets
        completed by parameter `tail_from` or later go out with `tail_config`."""
        tail = self.tail_config is not None and i >= self.tail_from
        for k in self._bucket_of_param[i]:
            self._pending[k] -= 1
            if self._pending[k] == 0:
                self._use(self.tail_config if tail else self.config)
                self.stats.tail += int(tail)
                self._launch(k, stream)

    def _launch(self, k: int, stream):
        b = self.bucket(k)
        self._works.append(self.comm.allreduce(b, async_op=True, stream=stream))
        self.stats.launched += 1
        self.stats.bytes += b.numel() * b.element_size()

    def finish(self, stream=None):
        """Make `stream` wait for every launched bucket (no host block)."""
        for w in self._works:
            w.wait(stream=stream)
        self._works = []
        if any(p != 0 for p in self._pending):
            raise RuntimeError("finish() before every gradient was marked ready")
        self.reset()
