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
PAPER.md:375, an SM-driven allreduce is not free — DESIGN.md §6); algo "ce"
moves the bytes with the copy engines instead (only a local fold on the SMs).

A virtual comm (n ranks on one GPU, hfr_init_virtual) gets one arena per
virtual rank and reduces each bucket across them with one
hfr_allreduce_virtual: the same kernels and bucket plan as one rank per GPU,
so the bucketed path is parity-tested on a single B200.

Configs.  `config` (the overlapped buckets) and `tail_config` (the buckets
completed by the last gradient GEMM, with nothing left to hide behind) are
full hfr configs; build them from the comm's own with
`HaiScaleDDP.derive(comm, max_ctas=..., ...)` (= dataclasses.replace of
comm.config) so the gradient scale carries over.  A config whose scale
differs from the comm's raises instead of silently summing where the caller
averages.  finish() restores the comm's config.

Measured on 4 B200s with a 7e9-parameter LLaMA-shaped backward (C5, median
of 15 interleaved repetitions, profiles/r02/c5_ddp_r02r_3x_n4.jsonl): the
best bit-exact setting by the step time (backward + exposed allreduce) is
FLAT with derive(comm, max_ctas=32, threads=256, stream_gate=1,
flat_staging=1) — register-staged comm CTAs (no shared memory) that share
SMs with the GEMM CTAs — plus a full-width tail_config: 1.05x the backward
alone, 0.82 of the full-width allreduce time hidden (3 runs: 0.817, 0.819,
0.821).  threads=128 throttles the comm further (overlap 0.87-0.88 against
its own, longer allreduce time, 0.76-0.79 against the full-width one, and a
1 ms longer step).  algo "nvls" (order-relaxed) with 16 CTAs: 0.85 of the
full-width time, 1.045x.
"""
from __future__ import annotations

import dataclasses
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
    """Gradient arena + asynchronous bucketed allreduce for one rank (or all
    virtual ranks of a virtual comm).

    Usage per step:
        ddp.zero_grad()                     (optional; the backward may overwrite instead)
        for i in backward order: write ddp.grad(i); ddp.mark_ready(i, stream)
        ddp.finish(stream)                  (stream waits for every bucket)
    grad(i) / bucket(k) are tensors for a real comm and lists of tensors (one
    per virtual rank) for a virtual comm.
    """

    @staticmethod
    def derive(comm, **changes):
        """comm.config with `changes` applied (keeps scale, timeout, ...)."""
        return dataclasses.replace(comm.config, **changes)

    def __init__(self, comm, numels: Sequence[int], dtype, bucket_bytes: int = 64 << 20,
                 config=None, tail_config=None, tail_from: Optional[int] = None):
        """`config`: the comm config for buckets that overlap the backward
        (e.g. few small CTAs); `tail_config`: the config for the buckets
        completed by marking parameter `tail_from` (backward order) or a later
        one — the last gradient GEMM of the step; nothing is left to overlap
        them with, so they may take the whole GPU.  tail_from None: the last
        parameter.  None configs: the comm's config.  Every rank makes the
        same choice for the same bucket (collective contract, include/hfr.h)."""
        import torch
        base = comm.config
        for name, cfg in (("config", config), ("tail_config", tail_config)):
            if cfg is not None and cfg.scale != base.scale:
                raise ValueError(f"{name}.scale={cfg.scale} differs from the comm's scale {base.scale}: build it "
                                 "with HaiScaleDDP.derive(comm, ...) (or set the comm's scale first)")
        self.comm = comm
        self.base = base
        self.config = config
        self.tail_config = tail_config
        self.tail_from = len(numels) - 1 if tail_from is None else tail_from
        self.dtype = dtype
        esz = torch.tensor([], dtype=dtype).element_size()
        self.bucket_elems = max(1, bucket_bytes // esz)
        self.param_ranges, self.bucket_ranges, self.bucket_params = plan_buckets(list(numels), self.bucket_elems)
        self.total = self.param_ranges[-1][1] if self.param_ranges else 0
        arena = comm.empty(max(1, self.total), dtype)
        self.virtual = isinstance(arena, list)
        self.arenas = arena if self.virtual else [arena]
        self.arena = arena
        self._pending = [len(m) for m in self.bucket_params]
        self._active = None
        self._bucket_of_param: List[List[int]] = [[] for _ in numels]
        for k, mem in enumerate(self.bucket_params):
            for i in mem:
                self._bucket_of_param[i].append(k)
        self._works = []
        self.stats = BucketStats()

    def zero_grad(self):
        for a in self.arenas:
            a.zero_()

    def _view(self, s: int, e: int):
        views = [a[s:e] for a in self.arenas]
        return views if self.virtual else views[0]

    def grad(self, i: int):
        return self._view(*self.param_ranges[i])

    def bucket(self, k: int):
        return self._view(*self.bucket_ranges[k])

    def reset(self):
        self._pending = [len(m) for m in self.bucket_params]
        self._works = []
        self._active = None  # re-apply the configs each step (the caller may have changed the comm's)

    def _use(self, cfg):
        cfg = cfg if cfg is not None else self.base
        if cfg is not self._active:
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
                if self.config is not None or self.tail_config is not None:
                    self._use(self.tail_config if tail else self.config)
                self.stats.tail += int(tail)
                self._launch(k, stream)

    def _launch(self, k: int, stream):
        b = self.bucket(k)
        if self.virtual:
            w = self.comm.allreduce_virtual(b, async_op=True, stream=stream)
            nbytes = b[0].numel() * b[0].element_size()
        else:
            w = self.comm.allreduce(b, async_op=True, stream=stream)
            nbytes = b.numel() * b.element_size()
        self._works.append(w)
        self.stats.launched += 1
        self.stats.bytes += nbytes

    def finish(self, stream=None):
        """Make `stream` wait for every launched bucket (no host block) and
        restore the comm's own config."""
        for w in self._works:
            w.wait(stream=stream)
        self._works = []
        if any(p != 0 for p in self._pending):
            raise RuntimeError("finish() before every gradient was marked ready")
        if self._active is not None and self._active is not self.base:
            self.comm.set_config(self.base)
        self.reset()
