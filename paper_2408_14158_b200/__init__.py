"""B200-native HFReduce (arXiv 2408.14158 §4) — thin Python binding over libhfr.so.

Argument marshalling only: every step of the allreduce runs in libhfr.so's
sm_100a kernels (include/hfr.h).  PyTorch provides device memory, streams and
the process group used once, at setup, to exchange CUDA IPC handles.  There is
no CPU or eager-PyTorch fallback: if the extension is missing every call raises.

    import paper_2408_14158_b200 as hfr
    comm = hfr.Comm.init()                      # one process per GPU (torchrun)
    g = comm.empty(n, torch.bfloat16)           # symmetric (zero-copy) memory
    work = comm.allreduce(g, async_op=True)     # HaiScale-style async
    work.wait()                                 # stream-ordered completion
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional, Sequence

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libhfr.so")  # the in-tree build; a missing file raises

SUCCESS, ERR_INVALID_ARGUMENT, ERR_UNSUPPORTED, ERR_CUDA, ERR_OUT_OF_MEMORY, ERR_PROTOCOL, \
    ERR_TIMEOUT, ERR_NOT_INITIALIZED, ERR_INTERNAL = range(9)
ALGO_AUTO, ALGO_FLAT, ALGO_DBT, ALGO_PAIR_DBT, ALGO_ONESHOT, ALGO_CE, ALGO_NVLS = range(7)
ALGOS = {"auto": ALGO_AUTO, "flat": ALGO_FLAT, "dbt": ALGO_DBT, "pair_dbt": ALGO_PAIR_DBT, "oneshot": ALGO_ONESHOT,
         "ce": ALGO_CE, "nvls": ALGO_NVLS}
FLOAT32, BFLOAT16, FLOAT16, FP8_E4M3, FP8_E5M2 = 0, 1, 2, 3, 4
SUM = 0
ALLREDUCE, REDUCE_SCATTER, ALLGATHER, REDUCE, BROADCAST = range(5)
COLLS = {"allreduce": ALLREDUCE, "reduce_scatter": REDUCE_SCATTER, "allgather": ALLGATHER, "reduce": REDUCE,
         "broadcast": BROADCAST}

# every symbol include/hfr.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "hfr_config_default", "hfr_init", "hfr_init_virtual", "hfr_comm_set_config",
    "hfr_comm_local_ranks", "hfr_comm_rank", "hfr_comm_nranks", "hfr_mem_alloc", "hfr_mem_free",
    "hfr_register", "hfr_deregister", "hfr_allreduce", "hfr_allreduce_virtual", "hfr_wait", "hfr_comm_status",
    "hfr_barrier", "hfr_finalize", "hfr_tree_query", "hfr_comm_launches", "hfr_status_string",
    "hfr_last_cuda_error", "hfr_set_trace", "hfr_collective", "hfr_collective_virtual", "hfr_shard_range",
)


class HfrError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        msg = f"{what}: {status_string(status)} ({status})"
        if status == ERR_CUDA:
            msg += f" [{_lib().hfr_last_cuda_error().decode()}]"
        super().__init__(msg)


class _Config(ctypes.Structure):
    _fields_ = [("algo", ctypes.c_int), ("chunk_elems", ctypes.c_size_t), ("max_ctas", ctypes.c_int),
                ("threads", ctypes.c_int), ("scale", ctypes.c_float), ("scratch_bytes", ctypes.c_size_t),
                ("timeout_ms", ctypes.c_int), ("oneshot_max_bytes", ctypes.c_size_t), ("stream_gate", ctypes.c_int),
                ("nvls_bytes", ctypes.c_size_t), ("flat_staging", ctypes.c_int), ("ll_push_max", ctypes.c_size_t),
                ("pdl_off", ctypes.c_int), ("tree_staging", ctypes.c_int)]


@dataclass
class Config:
    """Mirror of hfr_config_t (include/hfr.h); 0 means the library default."""
    algo: str = "auto"
    chunk_elems: int = 0
    max_ctas: int = 0
    threads: int = 0
    scale: float = 1.0
    scratch_bytes: int = 0
    timeout_ms: int = 0
    oneshot_max_bytes: int = 0
    stream_gate: int = 0
    nvls_bytes: int = 0
    flat_staging: int = 0
    ll_push_max: int = 0
    pdl_off: int = 0
    tree_staging: int = 0

    def _c(self) -> _Config:
        if self.algo not in ALGOS:
            raise ValueError(f"unknown algo {self.algo!r}")
        return _Config(ALGOS[self.algo], self.chunk_elems, self.max_ctas, self.threads, self.scale,
                       self.scratch_bytes, self.timeout_ms, self.oneshot_max_bytes, self.stream_gate,
                       self.nvls_bytes, self.flat_staging, self.ll_push_max, self.pdl_off,
                       self.tree_staging)


_LIB = None
_AG_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)


def _lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libhfr.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; "
                               "g.build()'` (nvcc, sm_100a). There is no fallback path.")
        L = ctypes.CDLL(LIB_PATH)
        vp, sz, i, p = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER
        sig = {
            "hfr_config_default": (None, [p(_Config)]),
            "hfr_init": (i, [p(vp), i, i, i, _AG_FN, vp, p(_Config)]),
            "hfr_init_virtual": (i, [p(vp), i, i, p(_Config)]),
            "hfr_comm_set_config": (i, [vp, p(_Config)]),
            "hfr_comm_local_ranks": (i, [vp]),
            "hfr_comm_rank": (i, [vp]),
            "hfr_comm_nranks": (i, [vp]),
            "hfr_mem_alloc": (i, [vp, sz, p(vp)]),
            "hfr_mem_free": (i, [vp, vp]),
            "hfr_register": (i, [vp, vp, sz]),
            "hfr_deregister": (i, [vp, vp]),
            "hfr_allreduce": (i, [vp, vp, sz, i, i, vp, p(vp)]),
            "hfr_allreduce_virtual": (i, [vp, p(vp), sz, i, i, vp, p(vp)]),
            "hfr_wait": (i, [vp, vp]),
            "hfr_comm_status": (i, [vp]),
            "hfr_barrier": (i, [vp, vp]),
            "hfr_finalize": (i, [vp]),
            "hfr_tree_query": (i, [i, i, p(i), p(i), p(i)]),
            "hfr_comm_launches": (ctypes.c_uint64, [vp]),
            "hfr_status_string": (ctypes.c_char_p, [i]),
            "hfr_last_cuda_error": (ctypes.c_char_p, []),
            "hfr_set_trace": (i, [vp, vp, sz]),
            "hfr_collective": (i, [vp, i, vp, sz, i, i, i, vp, p(vp)]),
            "hfr_collective_virtual": (i, [vp, i, p(vp), sz, i, i, i, vp, p(vp)]),
            "hfr_shard_range": (i, [i, sz, i, i, p(sz), p(sz)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def lib():
    """The loaded libhfr.so (ctypes.CDLL)."""
    return _lib()


def status_string(status: int) -> str:
    return _lib().hfr_status_string(status).decode()


def _check(status: int, what: str):
    if status != SUCCESS:
        raise HfrError(status, what)


def tree_query(n: int, which: int):
    """(parent, children) of double binary tree `which` (0=A, 1=B) over n ranks
    as libhfr builds it (reading R9) — host only, no GPU."""
    P = (ctypes.c_int * n)()
    C0 = (ctypes.c_int * n)()
    C1 = (ctypes.c_int * n)()
    _check(_lib().hfr_tree_query(n, which, P, C0, C1), "hfr_tree_query")
    children = [[c for c in (C0[v], C1[v]) if c >= 0] for v in range(n)]
    return list(P), children


def shard_range(nranks: int, count: int, dtype: str, rank: int):
    """[lo, hi) of rank's shard (hfr_shard_range; dtype 'f32' or 'bf16')."""
    lo, hi = ctypes.c_size_t(), ctypes.c_size_t()
    code = {"bf16": BFLOAT16, "bfloat16": BFLOAT16, "f16": FLOAT16, "float16": FLOAT16, "e4m3": FP8_E4M3,
            "e5m2": FP8_E5M2}.get(dtype, FLOAT32)
    _check(_lib().hfr_shard_range(nranks, count, code, rank, ctypes.byref(lo), ctypes.byref(hi)), "hfr_shard_range")
    return lo.value, hi.value


def _dtype_code(t) -> int:
    import torch
    if t.dtype == torch.float32:
        return FLOAT32
    if t.dtype == torch.bfloat16:
        return BFLOAT16
    if t.dtype == torch.float16:
        return FLOAT16
    if t.dtype == torch.float8_e4m3fn:
        return FP8_E4M3
    if t.dtype == torch.float8_e5m2:
        return FP8_E5M2
    raise TypeError(f"hfr supports float32, bfloat16, float16, float8_e4m3fn and float8_e5m2, not {t.dtype}")


def _stream_handle(stream) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


class _CudaBuf:
    """__cuda_array_interface__ view of library-owned device memory."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


class Work:
    """Handle of an asynchronous allreduce (hfr_req_t)."""

    def __init__(self, comm: "Comm", req: ctypes.c_void_p, keep):
        self._comm = comm
        self._req = req
        self._keep = keep  # tensors must stay alive until completion

    def wait(self, stream=None, host: bool = False):
        """Order completion onto `stream` (default: the current stream), or
        block the host when host=True (also surfaces PROTOCOL/TIMEOUT)."""
        if self._req is None:
            return
        if host:
            st = _lib().hfr_wait(self._req, None)
        else:
            h = _stream_handle(stream)
            st = _lib().hfr_wait(self._req, ctypes.c_void_p(h if h != 0 else 1))
        self._req = None
        self._keep = None
        _check(st, "hfr_wait")


def _torch_allgather(group):
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    world = dist.get_world_size(group)

    def ag(send, recv, nbytes, _ctx):
        try:
            src = torch.frombuffer(bytearray(ctypes.string_at(send, nbytes)), dtype=torch.uint8)
            if backend == "nccl":
                src = src.cuda()
            out = torch.empty(world * nbytes, dtype=torch.uint8, device=src.device)
            dist.all_gather_into_tensor(out, src, group=group)
            data = out.cpu().numpy().tobytes()
            ctypes.memmove(recv, data, len(data))
            return 0
        except Exception as e:  # noqa: BLE001 — report through the C status
            import sys
            print(f"hfr allgather callback failed: {e!r}", file=sys.stderr)
            return 1

    return ag


class Comm:
    """An HFReduce communicator (hfr_comm_t)."""

    def __init__(self, handle: ctypes.c_void_p, keepalive=None):
        self._h = handle
        self._keep = keepalive
        L = _lib()
        self.rank = L.hfr_comm_rank(handle)
        self.nranks = L.hfr_comm_nranks(handle)
        self.local_ranks = L.hfr_comm_local_ranks(handle)
        self.virtual = self.local_ranks > 1 or False
        self.config = Config()
        self._allocs = []

    # -- construction -------------------------------------------------------
    @classmethod
    def init(cls, group=None, device: Optional[int] = None, config: Optional[Config] = None) -> "Comm":
        """One rank per process over torch.distributed (COLLECTIVE)."""
        import torch
        import torch.distributed as dist
        rank = dist.get_rank(group)
        world = dist.get_world_size(group)
        if device is None:
            device = torch.cuda.current_device()
        cb = _AG_FN(_torch_allgather(group))
        h = ctypes.c_void_p()
        cfg = (config or Config())._c()
        _check(_lib().hfr_init(ctypes.byref(h), rank, world, device, cb, None, ctypes.byref(cfg)), "hfr_init")
        c = cls(h, keepalive=cb)
        c.virtual = False
        c.device = device
        c.config = config or Config()
        return c

    @classmethod
    def single(cls, device: int = 0, config: Optional[Config] = None) -> "Comm":
        """A real (one rank per process) comm with nranks = 1: no process
        group, no peers; every schedule reduces to scale-and-cast in place."""
        h = ctypes.c_void_p()
        cfg = (config or Config())._c()
        _check(_lib().hfr_init(ctypes.byref(h), 0, 1, device, _AG_FN(), None, ctypes.byref(cfg)), "hfr_init")
        c = cls(h)
        c.virtual = False
        c.device = device
        c.config = config or Config()
        return c

    @classmethod
    def virtual_ranks(cls, nranks: int, device: int = 0, config: Optional[Config] = None) -> "Comm":
        """n virtual ranks on one GPU (single process)."""
        h = ctypes.c_void_p()
        cfg = (config or Config())._c()
        _check(_lib().hfr_init_virtual(ctypes.byref(h), nranks, device, ctypes.byref(cfg)), "hfr_init_virtual")
        c = cls(h)
        c.virtual = True
        c.device = device
        c.config = config or Config()
        return c

    # -- configuration ------------------------------------------------------
    def set_config(self, config: Config):
        """Replace the whole configuration (COLLECTIVE; include/hfr.h
        hfr_comm_set_config).  `self.config` mirrors the current one; build
        variants with dataclasses.replace(comm.config, ...) to keep scale."""
        cfg = config._c()
        _check(_lib().hfr_comm_set_config(self._h, ctypes.byref(cfg)), "hfr_comm_set_config")
        self.config = config

    @property
    def launches(self) -> int:
        return int(_lib().hfr_comm_launches(self._h))

    def status(self) -> int:
        return _lib().hfr_comm_status(self._h)

    # -- memory ---------------------------------------------------------------
    def empty(self, numel: int, dtype):
        """Symmetric peer-mapped tensor(s) (COLLECTIVE): one tensor for a real
        comm, a list of local_ranks tensors for a virtual comm."""
        import torch
        esz = torch.tensor([], dtype=dtype).element_size()
        ptrs = (ctypes.c_void_p * self.local_ranks)()
        _check(_lib().hfr_mem_alloc(self._h, max(1, numel * esz), ptrs), "hfr_mem_alloc")
        out = []
        for p in ptrs:
            raw = torch.as_tensor(_CudaBuf(p, (max(1, numel * esz),), "|u1"), device=f"cuda:{self.device}")
            out.append(raw[: numel * esz].view(dtype))
        self._allocs.append(ptrs[0])
        return out if self.virtual else out[0]

    def free_all(self):
        """Release every allocation made with empty() (COLLECTIVE); tensors
        viewing them must not be used afterwards."""
        for p in self._allocs:
            _check(_lib().hfr_mem_free(self._h, ctypes.c_void_p(p)), "hfr_mem_free")
        self._allocs = []

    def register(self, tensor):
        """Make a cudaMalloc'ed tensor peer visible (COLLECTIVE) for zero-copy."""
        _check(_lib().hfr_register(self._h, ctypes.c_void_p(tensor.data_ptr()),
                                   tensor.numel() * tensor.element_size()), "hfr_register")

    def deregister(self, tensor):
        """Undo register() (COLLECTIVE); call before the memory is freed."""
        _check(_lib().hfr_deregister(self._h, ctypes.c_void_p(tensor.data_ptr())), "hfr_deregister")

    # -- collectives ---------------------------------------------------------
    def allreduce(self, tensor, async_op: bool = False, stream=None) -> Optional[Work]:
        """In-place sum-allreduce of a contiguous float32/bfloat16 CUDA tensor."""
        if self.virtual:
            raise ValueError("virtual comm: use allreduce_virtual(list_of_tensors)")
        if not tensor.is_contiguous():
            raise ValueError("tensor must be contiguous")
        req = ctypes.c_void_p()
        st = _lib().hfr_allreduce(self._h, ctypes.c_void_p(tensor.data_ptr()), tensor.numel(),
                                  _dtype_code(tensor), SUM, ctypes.c_void_p(_stream_handle(stream)),
                                  ctypes.byref(req) if async_op else None)
        _check(st, "hfr_allreduce")
        return Work(self, req, tensor) if async_op else None

    def allreduce_virtual(self, tensors: Sequence, async_op: bool = False, stream=None) -> Optional[Work]:
        """In-place allreduce over the virtual ranks' tensors (one per rank)."""
        if not self.virtual:
            raise ValueError("not a virtual comm")
        if len(tensors) != self.nranks:
            raise ValueError(f"need {self.nranks} tensors")
        t0 = tensors[0]
        for t in tensors:
            if t.numel() != t0.numel() or t.dtype != t0.dtype or not t.is_contiguous():
                raise ValueError("tensors must match in numel/dtype and be contiguous")
        ptrs = (ctypes.c_void_p * self.nranks)(*[t.data_ptr() for t in tensors])
        req = ctypes.c_void_p()
        st = _lib().hfr_allreduce_virtual(self._h, ptrs, t0.numel(), _dtype_code(t0), SUM,
                                          ctypes.c_void_p(_stream_handle(stream)),
                                          ctypes.byref(req) if async_op else None)
        _check(st, "hfr_allreduce_virtual")
        return Work(self, req, list(tensors)) if async_op else None

    def set_trace(self, buf=None):
        """Diagnostic chunk timelines of the tree schedules into a uint8 CUDA
        tensor (None: off).  See include/hfr.h hfr_set_trace."""
        if buf is None:
            _check(_lib().hfr_set_trace(self._h, None, 0), "hfr_set_trace")
        else:
            _check(_lib().hfr_set_trace(self._h, ctypes.c_void_p(buf.data_ptr()), buf.numel() * buf.element_size()),
                   "hfr_set_trace")

    def collective(self, kind: str, tensor, root: int = 0, async_op: bool = False, stream=None) -> Optional[Work]:
        """In-place collective (include/hfr.h hfr_collective): 'allreduce',
        'reduce_scatter', 'allgather', 'reduce', 'broadcast'."""
        if self.virtual:
            raise ValueError("virtual comm: use collective_virtual(kind, list_of_tensors)")
        if not tensor.is_contiguous():
            raise ValueError("tensor must be contiguous")
        req = ctypes.c_void_p()
        st = _lib().hfr_collective(self._h, COLLS[kind], ctypes.c_void_p(tensor.data_ptr()), tensor.numel(),
                                   _dtype_code(tensor), SUM, root, ctypes.c_void_p(_stream_handle(stream)),
                                   ctypes.byref(req) if async_op else None)
        _check(st, f"hfr_collective({kind})")
        return Work(self, req, tensor) if async_op else None

    def collective_virtual(self, kind: str, tensors: Sequence, root: int = 0, async_op: bool = False,
                           stream=None) -> Optional[Work]:
        if not self.virtual:
            raise ValueError("not a virtual comm")
        if len(tensors) != self.nranks:
            raise ValueError(f"need {self.nranks} tensors")
        t0 = tensors[0]
        for t in tensors:
            if t.numel() != t0.numel() or t.dtype != t0.dtype or not t.is_contiguous():
                raise ValueError("tensors must match in numel/dtype and be contiguous")
        ptrs = (ctypes.c_void_p * self.nranks)(*[t.data_ptr() for t in tensors])
        req = ctypes.c_void_p()
        st = _lib().hfr_collective_virtual(self._h, COLLS[kind], ptrs, t0.numel(), _dtype_code(t0), SUM, root,
                                           ctypes.c_void_p(_stream_handle(stream)),
                                           ctypes.byref(req) if async_op else None)
        _check(st, f"hfr_collective_virtual({kind})")
        return Work(self, req, list(tensors)) if async_op else None

    def barrier(self, stream=None):
        _check(_lib().hfr_barrier(self._h, ctypes.c_void_p(_stream_handle(stream))), "hfr_barrier")

    def finalize(self):
        if self._h:
            _check(_lib().hfr_finalize(self._h), "hfr_finalize")
            self._h = None


# -- module-level convenience (hfr.init(group), hfr.allreduce(t, async_op)) --
_default: Optional[Comm] = None


def init(group=None, device: Optional[int] = None, config: Optional[Config] = None) -> Comm:
    """COLLECTIVE.  Create the process's default communicator over `group`
    (torch.distributed; default group if None) and return it."""
    global _default
    if _default is not None:
        raise RuntimeError("hfr.init: already initialised (call hfr.finalize() first)")
    _default = Comm.init(group=group, device=device, config=config)
    return _default


def allreduce(tensor, async_op: bool = False, stream=None) -> Optional[Work]:
    """In-place sum-allreduce of `tensor` on the default communicator."""
    if _default is None:
        raise RuntimeError("hfr.allreduce: call hfr.init(group) first")
    return _default.allreduce(tensor, async_op=async_op, stream=stream)


def finalize() -> None:
    """COLLECTIVE.  Tear down the default communicator."""
    global _default
    if _default is not None:
        _default.finalize()
        _default = None


__all__ = ["Comm", "Config", "Work", "HfrError", "tree_query", "shard_range", "status_string", "lib", "LIB_PATH",
           "EXPORTS", "COLLS", "init", "allreduce", "finalize"]
