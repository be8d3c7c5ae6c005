"""B200-native unified-tensor gather (PyTorch-Direct, arXiv 2101.07956): Python binding.

Argument marshalling over the C ABI in ``include/ut.h`` (``libut.so``, built in-tree from
``csrc/``); every step of the gather runs in the library's sm_100a kernels. PyTorch supplies
device memory and streams only. There is no CPU fallback: if ``libut.so`` cannot be built or
loaded, importing the binding raises.

Low level (same names and arguments as the C ABI, raw addresses and ints):
    ut_register(host_addr, rows, row_bytes) -> handle
    ut_gather(handle, idx_dev_addr, n, out_dev_addr, stream_handle)
    ut_gather_host(handle, idx_host_addr, n, out_host_addr, stream_handle)
    ut_release(handle), ut_error_pos(handle, stream_handle) -> int, ut_get_stats(handle),
    ut_plan_name(handle), ut_set_plan(handle, name), ut_plan_probe(base, rows, rb, out),
    ut_table_get_info(handle) -> dict
    ut_coop_create / _export / _open / _dispatch / _fetch / _combine / _gather / _get_stats /
    _error_pos / _owner / _release (the cooperative multi-rank gather)
    ut_pool_create / _alloc / _free / _release_cached / _get_stats / _destroy / _table (the
    unified allocator with block recycling)

High level: ``Table`` — the paper's unified tensor, ``Table(features)[gpu_idx]`` being
``unified_tensor[gpu_tensor]``; ``Coop`` — one rank's side of the cooperative
gather (rows requested by several ranks cross the host link once); ``Graph`` — GPU sampling;
``Pool`` — the recycling unified allocator (``Table.from_pool``).
"""
from __future__ import annotations

import ctypes
import os

from . import _build

UT_OK, UT_EINVAL, UT_ENOMEM, UT_ECUDA, UT_ERANGE, UT_ENOTSUP = 0, -1, -2, -3, -4, -5

# Every symbol include/ut.h declares (tests check the library exports exactly these).
ABI = ("ut_register", "ut_gather", "ut_gather_host", "ut_release", "ut_error_pos",
       "ut_last_error", "ut_plan_name", "ut_plan_probe", "ut_set_plan", "ut_table_get_info",
       "ut_get_stats", "ut_create", "ut_graph_register", "ut_graph_set_option", "ut_sample",
       "ut_graph_release", "ut_mem_advise", "ut_gather_dn", "ut_sample_async",
       "ut_sample_capacity", "ut_graph_launches", "ut_coop_create", "ut_coop_export",
       "ut_coop_open", "ut_coop_dispatch", "ut_coop_fetch", "ut_coop_combine", "ut_coop_gather",
       "ut_coop_get_stats", "ut_coop_error_pos", "ut_coop_owner", "ut_coop_release",
       "ut_coop_create_partitioned", "ut_coop_partition_ids", "ut_coop_open_local",
       "ut_gather_multi", "ut_numa_interleave", "ut_gather_i32", "ut_numa_place",
       "ut_pool_create", "ut_pool_alloc", "ut_pool_free", "ut_pool_release_cached",
       "ut_pool_get_stats", "ut_pool_destroy", "ut_pool_table")

UT_COOP_HANDLE_BYTES = 64

UT_ALLOC = {"pinned": 0, "managed": 1, "vmm": 2, "system": 3}


class UTError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class _Info(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_uint64), ("row_bytes", ctypes.c_uint64),
                ("host_addr", ctypes.c_uint64), ("dev_addr", ctypes.c_uint64),
                ("registered", ctypes.c_int), ("alloc_kind", ctypes.c_int),
                ("read_only", ctypes.c_int),
                ("base_mod128", ctypes.c_int), ("device", ctypes.c_int)]


class _Stats(ctypes.Structure):
    _fields_ = [("gathers", ctypes.c_uint64), ("kernel_launches", ctypes.c_uint64),
                ("rows", ctypes.c_uint64), ("bytes", ctypes.c_uint64),
                ("timed_launches", ctypes.c_uint64), ("gather_kernel_ms", ctypes.c_double),
                ("share_gathers", ctypes.c_uint64)]


class _PoolStats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint64) for k in ("backend_calls", "backend_frees", "recycled_hits",
                                               "bytes_live", "bytes_cached", "blocks_live",
                                               "blocks_cached", "limit_bytes")]


class _CoopStats(ctypes.Structure):
    _fields_ = [("steps", ctypes.c_uint64), ("requested_rows", ctypes.c_uint64),
                ("owner_requests", ctypes.c_uint64), ("unique_rows_fetched", ctypes.c_uint64),
                ("last_unique_rows", ctypes.c_uint64), ("kernel_launches", ctypes.c_uint64),
                ("stream_memops", ctypes.c_uint64),
                ("block_rows", ctypes.c_uint64), ("region_bytes", ctypes.c_uint64)]


def _load():
    path = os.environ.get("UT_LIB") or _build.build()   # UT_LIB: an A/B build of the same source
    L = ctypes.CDLL(path)
    vp, u64, i64p = ctypes.c_void_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_int64)
    L.ut_register.restype = vp
    L.ut_register.argtypes = [vp, u64, u64]
    L.ut_gather.restype = ctypes.c_int
    L.ut_gather.argtypes = [vp, vp, u64, vp, vp]
    L.ut_gather_host.restype = ctypes.c_int
    L.ut_gather_host.argtypes = [vp, vp, u64, vp, vp]
    L.ut_release.restype = ctypes.c_int
    L.ut_release.argtypes = [vp]
    L.ut_error_pos.restype = ctypes.c_int
    L.ut_error_pos.argtypes = [vp, vp, i64p]
    L.ut_last_error.restype = ctypes.c_int
    L.ut_last_error.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
    L.ut_plan_name.restype = ctypes.c_char_p
    L.ut_plan_name.argtypes = [vp]
    L.ut_plan_probe.restype = ctypes.c_char_p
    L.ut_plan_probe.argtypes = [u64, u64, u64, u64]
    L.ut_set_plan.restype = ctypes.c_int
    L.ut_set_plan.argtypes = [vp, ctypes.c_char_p]
    L.ut_table_get_info.restype = ctypes.c_int
    L.ut_table_get_info.argtypes = [vp, ctypes.POINTER(_Info)]
    L.ut_create.restype = vp
    L.ut_create.argtypes = [vp, u64, u64, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
    L.ut_pool_create.restype = vp
    L.ut_pool_create.argtypes = [ctypes.c_int, u64]
    L.ut_pool_alloc.restype = ctypes.c_int
    L.ut_pool_alloc.argtypes = [vp, u64, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(u64)]
    L.ut_pool_free.restype = ctypes.c_int
    L.ut_pool_free.argtypes = [vp, vp]
    L.ut_pool_release_cached.restype = ctypes.c_int
    L.ut_pool_release_cached.argtypes = [vp]
    L.ut_pool_get_stats.restype = ctypes.c_int
    L.ut_pool_get_stats.argtypes = [vp, ctypes.POINTER(_PoolStats)]
    L.ut_pool_destroy.restype = ctypes.c_int
    L.ut_pool_destroy.argtypes = [vp]
    L.ut_pool_table.restype = vp
    L.ut_pool_table.argtypes = [vp, vp, u64, u64, ctypes.POINTER(ctypes.c_void_p)]
    L.ut_graph_register.restype = vp
    L.ut_graph_register.argtypes = [vp, vp, u64, u64]
    L.ut_graph_set_option.restype = ctypes.c_int
    L.ut_graph_set_option.argtypes = [vp, ctypes.c_char_p]
    L.ut_sample.restype = ctypes.c_int
    L.ut_sample.argtypes = [vp, vp, u64, vp, ctypes.c_int, u64, vp, u64,
                            ctypes.POINTER(ctypes.c_uint64), vp]
    L.ut_gather_multi.restype = ctypes.c_int
    L.ut_gather_multi.argtypes = [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(vp),
                                  ctypes.POINTER(u64), ctypes.POINTER(vp), ctypes.POINTER(vp)]
    L.ut_gather_i32.restype = ctypes.c_int
    L.ut_gather_i32.argtypes = [vp, vp, u64, vp, vp]
    L.ut_gather_dn.restype = ctypes.c_int
    L.ut_gather_dn.argtypes = [vp, vp, vp, u64, vp, vp]
    L.ut_sample_async.restype = ctypes.c_int
    L.ut_sample_async.argtypes = [vp, vp, u64, vp, ctypes.c_int, u64, vp, u64, vp, vp]
    L.ut_sample_capacity.restype = ctypes.c_uint64
    L.ut_sample_capacity.argtypes = [u64, vp, ctypes.c_int, u64]
    L.ut_graph_launches.restype = ctypes.c_uint64
    L.ut_graph_launches.argtypes = [vp]
    L.ut_mem_advise.restype = ctypes.c_int
    L.ut_mem_advise.argtypes = [vp, ctypes.c_int, ctypes.c_int]
    L.ut_numa_interleave.restype = ctypes.c_int
    L.ut_numa_interleave.argtypes = [vp, ctypes.c_int, u64]
    L.ut_numa_place.restype = ctypes.c_int
    L.ut_numa_place.argtypes = [vp, ctypes.c_int]
    L.ut_graph_release.restype = ctypes.c_int
    L.ut_graph_release.argtypes = [vp]
    L.ut_get_stats.restype = ctypes.c_int
    L.ut_get_stats.argtypes = [vp, ctypes.POINTER(_Stats), ctypes.c_int]
    L.ut_coop_create.restype = vp
    L.ut_coop_create.argtypes = [vp, ctypes.c_int, ctypes.c_int, u64]
    L.ut_coop_create_partitioned.restype = vp
    L.ut_coop_create_partitioned.argtypes = [vp, u64, ctypes.c_int, ctypes.c_int, u64]
    L.ut_coop_partition_ids.restype = ctypes.c_uint64
    L.ut_coop_partition_ids.argtypes = [u64, u64, ctypes.c_int, ctypes.c_int, vp, u64]
    L.ut_coop_export.restype = ctypes.c_int
    L.ut_coop_export.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_uint64)]
    L.ut_coop_open.restype = ctypes.c_int
    L.ut_coop_open.argtypes = [vp, vp]
    L.ut_coop_open_local.restype = ctypes.c_int
    L.ut_coop_open_local.argtypes = [vp, ctypes.POINTER(vp), ctypes.c_int]
    L.ut_coop_dispatch.restype = ctypes.c_int
    L.ut_coop_dispatch.argtypes = [vp, vp, u64, vp]
    L.ut_coop_fetch.restype = ctypes.c_int
    L.ut_coop_fetch.argtypes = [vp, vp]
    L.ut_coop_combine.restype = ctypes.c_int
    L.ut_coop_combine.argtypes = [vp, vp, vp]
    L.ut_coop_gather.restype = ctypes.c_int
    L.ut_coop_gather.argtypes = [vp, vp, u64, vp, vp]
    L.ut_coop_get_stats.restype = ctypes.c_int
    L.ut_coop_get_stats.argtypes = [vp, ctypes.POINTER(_CoopStats)]
    L.ut_coop_error_pos.restype = ctypes.c_int
    L.ut_coop_error_pos.argtypes = [vp, vp, i64p]
    L.ut_coop_owner.restype = ctypes.c_uint32
    L.ut_coop_owner.argtypes = [u64, u64, ctypes.c_int, ctypes.c_int64, ctypes.POINTER(ctypes.c_uint64)]
    L.ut_coop_release.restype = ctypes.c_int
    L.ut_coop_release.argtypes = [vp]
    return L


_lib = _load()
LIB_PATH = os.environ.get("UT_LIB") or _build.LIB


def last_error() -> tuple[int, str]:
    buf = ctypes.create_string_buffer(512)
    code = _lib.ut_last_error(buf, 512)
    return code, buf.value.decode(errors="replace")


def _check(rc: int) -> int:
    if rc != UT_OK:
        code, msg = last_error()
        raise UTError(rc, msg)
    return rc


# ---- the C ABI, name for name ---------------------------------------------------------------
def ut_register(host_addr: int, rows: int, row_bytes: int) -> int:
    h = _lib.ut_register(host_addr, rows, row_bytes)
    if not h:
        code, msg = last_error()
        raise UTError(code, msg)
    return h


def ut_create(src: int, rows: int, row_bytes: int, kind: int) -> tuple[int, int]:
    """(handle, host address) of a new library-owned table (src 0/None: left for the caller)."""
    host = ctypes.c_void_p()
    h = _lib.ut_create(src or None, rows, row_bytes, kind, ctypes.byref(host))
    if not h:
        code, msg = last_error()
        raise UTError(code, msg)
    return h, int(host.value)


def ut_pool_create(kind: int, limit_bytes: int = 0) -> int:
    h = _lib.ut_pool_create(kind, limit_bytes)
    if not h:
        code, msg = last_error()
        raise UTError(code, msg)
    return h


def ut_pool_alloc(p: int, nbytes: int) -> tuple[int, int]:
    """(host address or 0, capacity) of a pool block."""
    host, cap = ctypes.c_void_p(), ctypes.c_uint64()
    _check(_lib.ut_pool_alloc(p, nbytes, ctypes.byref(host), ctypes.byref(cap)))
    return int(host.value or 0), int(cap.value)


def ut_pool_free(p: int, host: int) -> None:
    _check(_lib.ut_pool_free(p, host or None))


def ut_pool_release_cached(p: int) -> None:
    _check(_lib.ut_pool_release_cached(p))


def ut_pool_get_stats(p: int) -> dict:
    st = _PoolStats()
    _check(_lib.ut_pool_get_stats(p, ctypes.byref(st)))
    return {k: getattr(st, k) for k, _ in st._fields_}


def ut_pool_destroy(p: int) -> None:
    _check(_lib.ut_pool_destroy(p))


def ut_pool_table(p: int, src: int, rows: int, row_bytes: int) -> tuple[int, int]:
    """(handle, host address) of a table over a pool block; ut_release gives the block back."""
    host = ctypes.c_void_p()
    h = _lib.ut_pool_table(p, src or None, rows, row_bytes, ctypes.byref(host))
    if not h:
        code, msg = last_error()
        raise UTError(code, msg)
    return h, int(host.value)


def ut_gather(t: int, idx_dev: int, n: int, out_dev: int, stream: int = 0) -> None:
    _check(_lib.ut_gather(t, idx_dev, n, out_dev, stream))


def ut_gather_i32(t: int, idx_dev: int, n: int, out_dev: int, stream: int = 0) -> None:
    _check(_lib.ut_gather_i32(t, idx_dev, n, out_dev, stream))


def ut_gather_host(t: int, idx_host: int, n: int, out_host: int, stream: int = 0) -> None:
    _check(_lib.ut_gather_host(t, idx_host, n, out_host, stream))


def ut_release(t: int) -> None:
    _check(_lib.ut_release(t))


def ut_error_pos(t: int, stream: int = 0) -> int:
    v = ctypes.c_int64(-1)
    rc = _lib.ut_error_pos(t, stream, ctypes.byref(v))
    if rc not in (UT_OK, UT_ERANGE):
        _check(rc)
    return int(v.value)


def ut_plan_name(t: int) -> str:
    return _lib.ut_plan_name(t).decode()


def ut_plan_probe(base: int, rows: int, row_bytes: int, out: int = 0) -> str:
    return _lib.ut_plan_probe(base, rows, row_bytes, out).decode()


def ut_set_plan(t: int, name: str) -> None:
    _check(_lib.ut_set_plan(t, name.encode()))


def ut_table_get_info(t: int) -> dict:
    info = _Info()
    _check(_lib.ut_table_get_info(t, ctypes.byref(info)))
    return {k: getattr(info, k) for k, _ in _Info._fields_}


def ut_get_stats(t: int, reset: bool = False) -> dict:
    st = _Stats()
    _check(_lib.ut_get_stats(t, ctypes.byref(st), 1 if reset else 0))
    return {k: getattr(st, k) for k, _ in _Stats._fields_}


def ut_graph_register(indptr_addr: int, indices_addr: int, n_nodes: int, n_edges: int) -> int:
    h = _lib.ut_graph_register(indptr_addr, indices_addr, n_nodes, n_edges)
    if not h:
        code, msg = last_error()
        raise UTError(code, msg)
    return h


def ut_graph_set_option(g: int, option: str) -> None:
    _check(_lib.ut_graph_set_option(g, option.encode()))


def ut_sample(g: int, seeds_dev: int, n_seeds: int, fanouts, seed: int, nodes_dev: int, cap: int,
              stream: int = 0) -> int:
    fan = (ctypes.c_int32 * len(fanouts))(*fanouts)
    n = ctypes.c_uint64(0)
    rc = _lib.ut_sample(g, seeds_dev, n_seeds, fan, len(fanouts), seed & 0xFFFFFFFFFFFFFFFF,
                        nodes_dev, cap, ctypes.byref(n), stream)
    if rc != UT_OK:
        code, msg = last_error()
        raise UTError(rc, msg)
    return int(n.value)


def ut_mem_advise(t: int, advice: int, device: int) -> int:
    """cudaMemAdvise on the table's storage; returns the CUDA error code (0 = success)."""
    rc = _lib.ut_mem_advise(t, advice, device)
    if rc < 0:
        _check(rc)
    return rc


def ut_numa_interleave(t: int, nodes: int, chunk_bytes: int = 0) -> None:
    """Stripe a managed table's pages over host NUMA nodes 0..nodes-1 (before it is filled)."""
    _check(_lib.ut_numa_interleave(t, nodes, chunk_bytes))


def ut_numa_place(t: int, node: int) -> None:
    """Put a whole managed table on one host NUMA node (before it is filled)."""
    _check(_lib.ut_numa_place(t, node))


def ut_gather_multi(t: int, devs: list[int], idx_dev: list[int], n: list[int], out_dev: list[int],
                    streams: list[int] | None = None) -> None:
    k = len(devs)
    assert len(idx_dev) == k and len(n) == k and len(out_dev) == k
    VP = ctypes.c_void_p * k
    st = VP(*(streams or [0] * k))
    _check(_lib.ut_gather_multi(t, k, (ctypes.c_int * k)(*devs), VP(*idx_dev),
                                (ctypes.c_uint64 * k)(*n), VP(*out_dev), st))


def ut_gather_dn(t: int, idx_dev: int, n_dev: int, max_n: int, out_dev: int, stream: int = 0) -> None:
    _check(_lib.ut_gather_dn(t, idx_dev, n_dev, max_n, out_dev, stream))


def ut_sample_capacity(n_seeds: int, fanouts, n_nodes: int) -> int:
    fan = (ctypes.c_int32 * max(1, len(fanouts)))(*fanouts)
    return int(_lib.ut_sample_capacity(n_seeds, fan, len(fanouts), n_nodes))


def ut_sample_async(g: int, seeds_dev: int, n_seeds: int, fanouts, seed: int, nodes_dev: int,
                    cap: int, n_out_dev: int, stream: int = 0) -> None:
    fan = (ctypes.c_int32 * max(1, len(fanouts)))(*fanouts)
    _check(_lib.ut_sample_async(g, seeds_dev, n_seeds, fan, len(fanouts),
                                seed & 0xFFFFFFFFFFFFFFFF, nodes_dev, cap, n_out_dev, stream))


def ut_graph_release(g: int) -> None:
    _check(_lib.ut_graph_release(g))


def ut_coop_create(t: int, world: int, rank: int, max_n: int) -> int:
    h = _lib.ut_coop_create(t, world, rank, max_n)
    if not h:
        code, msg = last_error()
        raise UTError(code, msg)
    return h


def ut_coop_create_partitioned(part: int, rows: int, world: int, rank: int, max_n: int) -> int:
    h = _lib.ut_coop_create_partitioned(part, rows, world, rank, max_n)
    if not h:
        code, msg = last_error()
        raise UTError(code, msg)
    return h


def ut_coop_partition_ids(rows: int, row_bytes: int, world: int, rank: int):
    """int64 numpy array: the table row of each local row of `rank`'s partition (-1 = padding)."""
    import numpy as np
    k = int(_lib.ut_coop_partition_ids(rows, row_bytes, world, rank, None, 0))
    ids = np.empty(k, dtype=np.int64)
    if k:
        _lib.ut_coop_partition_ids(rows, row_bytes, world, rank, ids.ctypes.data, k)
    return ids


def ut_coop_export(c: int) -> bytes:
    buf = ctypes.create_string_buffer(UT_COOP_HANDLE_BYTES)
    _check(_lib.ut_coop_export(c, buf, None))
    return buf.raw


def ut_coop_open(c: int, handles: bytes) -> None:
    _check(_lib.ut_coop_open(c, handles))


def ut_coop_open_local(c: int, peers: list[int]) -> None:
    arr = (ctypes.c_void_p * len(peers))(*peers)
    _check(_lib.ut_coop_open_local(c, arr, len(peers)))


def ut_coop_dispatch(c: int, idx_dev: int, n: int, stream: int = 0) -> None:
    _check(_lib.ut_coop_dispatch(c, idx_dev, n, stream))


def ut_coop_fetch(c: int, stream: int = 0) -> None:
    _check(_lib.ut_coop_fetch(c, stream))


def ut_coop_combine(c: int, out_dev: int, stream: int = 0) -> None:
    _check(_lib.ut_coop_combine(c, out_dev, stream))


def ut_coop_gather(c: int, idx_dev: int, n: int, out_dev: int, stream: int = 0) -> None:
    _check(_lib.ut_coop_gather(c, idx_dev, n, out_dev, stream))


def ut_coop_get_stats(c: int) -> dict:
    st = _CoopStats()
    _check(_lib.ut_coop_get_stats(c, ctypes.byref(st)))
    return {k: getattr(st, k) for k, _ in _CoopStats._fields_}


def ut_coop_error_pos(c: int, stream: int = 0) -> int:
    v = ctypes.c_int64(-1)
    rc = _lib.ut_coop_error_pos(c, stream, ctypes.byref(v))
    if rc not in (UT_OK, UT_ERANGE):
        _check(rc)
    return int(v.value)


def ut_coop_owner(rows: int, row_bytes: int, world: int, row_id: int) -> tuple[int, int]:
    """(owner rank, local index) of a row; (2**32 - 1, 0) for invalid arguments."""
    loc = ctypes.c_uint64(0)
    o = _lib.ut_coop_owner(rows, row_bytes, world, row_id, ctypes.byref(loc))
    return int(o), int(loc.value)


def ut_coop_release(c: int) -> None:
    _check(_lib.ut_coop_release(c))


# ---- convenience ----------------------------------------------------------------------------
def _stream_handle(stream) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


class Table:
    """A host-resident feature table that GPU kernels read directly (the "unified tensor").

    ``host`` is a numpy array or CPU torch tensor (any dtype; its rows are the table rows), or a
    raw address with ``rows`` and ``row_bytes``. The memory is pinned and mapped in place by
    ``ut_register`` (no copy) and must outlive the Table."""

    def __init__(self, host, rows: int | None = None, row_bytes: int | None = None):
        self._keep = host
        if isinstance(host, int):
            assert rows is not None and row_bytes is not None
            addr = host
        else:
            if hasattr(host, "data_ptr"):        # torch tensor
                assert not host.is_cuda and host.is_contiguous()
                addr = host.data_ptr()
                nbytes = host.numel() * host.element_size()
                shape = tuple(host.shape)
            else:                                 # numpy
                assert host.flags.c_contiguous
                addr = host.ctypes.data
                nbytes = host.nbytes
                shape = host.shape
            if rows is None:
                rows = shape[0] if len(shape) > 1 else nbytes
            if row_bytes is None:
                row_bytes = nbytes // rows
        self.rows, self.row_bytes, self.host_addr = int(rows), int(row_bytes), int(addr)
        self.handle = ut_register(self.host_addr, self.rows, self.row_bytes)

    @classmethod
    def create(cls, rows: int, row_bytes: int, kind: str = "pinned", src=None) -> "Table":
        """The paper's `to("unified")`: a new host-resident table of `kind` ("pinned",
        "managed" or "vmm") owned by the library; fill it through `.array()` or copy `src`."""
        addr = None
        if src is not None:
            addr = src.ctypes.data if hasattr(src, "ctypes") else src.data_ptr()
        self = cls.__new__(cls)
        self._keep = src
        self.handle, self.host_addr = ut_create(addr, rows, row_bytes, UT_ALLOC[kind])
        self.rows, self.row_bytes = int(rows), int(row_bytes)
        return self

    @classmethod
    def from_pool(cls, pool: "Pool", rows: int, row_bytes: int, src=None) -> "Table":
        """`Table.create` over a block of `pool` (the recycling unified allocator):
        closing the table caches the block in the pool instead of freeing it."""
        addr = None
        if src is not None:
            addr = src.ctypes.data if hasattr(src, "ctypes") else src.data_ptr()
        self = cls.__new__(cls)
        self._keep = (src, pool)                # the pool outlives its tables
        self.handle, self.host_addr = ut_pool_table(pool.handle, addr, rows, row_bytes)
        self.rows, self.row_bytes = int(rows), int(row_bytes)
        return self

    def array(self):
        """uint8 numpy view of the table's host bytes (no copy)."""
        import numpy as np
        buf = (ctypes.c_uint8 * (self.rows * self.row_bytes)).from_address(self.host_addr)
        return np.ctypeslib.as_array(buf)

    @property
    def plan(self) -> str:
        return ut_plan_name(self.handle)

    def set_plan(self, name: str) -> None:
        ut_set_plan(self.handle, name)

    def info(self) -> dict:
        return ut_table_get_info(self.handle)

    def numa_interleave(self, nodes: int, chunk_bytes: int = 0) -> None:
        """Managed tables: host pages striped over NUMA nodes 0..nodes-1 (call before filling)."""
        ut_numa_interleave(self.handle, nodes, chunk_bytes)

    def numa_place(self, node: int) -> None:
        """Managed tables: every host page on NUMA node `node` (call before filling)."""
        ut_numa_place(self.handle, node)

    def stats(self, reset: bool = False) -> dict:
        return ut_get_stats(self.handle, reset)

    def gather(self, idx, out=None, stream=None):
        """out[i] = row idx[i] (uint8 [n, row_bytes] CUDA tensor); idx: CUDA int64 (or int32)
        tensor."""
        import torch
        assert idx.is_cuda and idx.dtype in (torch.int64, torch.int32) and idx.is_contiguous()
        n = idx.numel()
        if out is None:
            out = torch.empty((n, self.row_bytes), dtype=torch.uint8, device=idx.device)
        else:
            assert out.is_cuda and out.is_contiguous()
            assert out.numel() * out.element_size() >= n * self.row_bytes
            assert out.device == idx.device
        go = ut_gather if idx.dtype == torch.int64 else ut_gather_i32
        # the C ABI gathers on the CURRENT device: make it the one idx and out live on, whatever
        # the caller's current device is (and take that device's current stream by default)
        with torch.cuda.device(idx.device):
            go(self.handle, idx.data_ptr(), n, out.data_ptr(),
               _stream_handle(stream if stream is not None else torch.cuda.current_stream(idx.device)))
        return out

    __getitem__ = gather

    def gather_multi(self, idxs, outs=None, streams=None):
        """The box form (ut_gather_multi): idxs[k] is a CUDA int64 tensor on any device; one
        call enqueues every device's gather from this thread. Returns the outputs."""
        import torch
        if outs is None:
            outs = [torch.empty((i.numel(), self.row_bytes), dtype=torch.uint8, device=i.device)
                    for i in idxs]
        for i, o in zip(idxs, outs):
            assert i.is_cuda and i.dtype == torch.int64 and i.is_contiguous()
            assert o.device == i.device and o.numel() * o.element_size() >= i.numel() * self.row_bytes
        sts = [_stream_handle(s) for s in streams] if streams is not None else \
              [int(torch.cuda.current_stream(i.device).cuda_stream) for i in idxs]
        ut_gather_multi(self.handle, [i.device.index for i in idxs], [i.data_ptr() for i in idxs],
                        [i.numel() for i in idxs], [o.data_ptr() for o in outs], sts)
        return outs

    def gather_dn(self, idx, n_dev, out, stream=None):
        """Gather min(n_dev[0], idx.numel()) rows; the count is read on the device."""
        import torch
        assert idx.device == n_dev.device == out.device
        with torch.cuda.device(idx.device):
            ut_gather_dn(self.handle, idx.data_ptr(), n_dev.data_ptr(), idx.numel(), out.data_ptr(),
                         _stream_handle(stream if stream is not None else torch.cuda.current_stream(idx.device)))
        return out

    def gather_host(self, idx_host, out_host=None, stream=None):
        """End-to-end form: host int64 idx in, host rows out (uint8 [n, row_bytes])."""
        import torch
        if not hasattr(idx_host, "data_ptr"):
            idx_host = torch.from_numpy(idx_host)
        assert not idx_host.is_cuda and idx_host.dtype == torch.int64 and idx_host.is_contiguous()
        n = idx_host.numel()
        if out_host is None:
            out_host = torch.empty((n, self.row_bytes), dtype=torch.uint8, pin_memory=True)
        ut_gather_host(self.handle, idx_host.data_ptr(), n, out_host.data_ptr(),
                       _stream_handle(stream))
        return out_host

    def error_pos(self, stream=None) -> int:
        """First out-of-range position since the last call (syncs the stream), or -1."""
        return ut_error_pos(self.handle, _stream_handle(stream))

    def close(self) -> None:
        if getattr(self, "handle", None):
            ut_release(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Pool:
    """The unified allocator with block recycling (``ut_pool_*``): host
    blocks of one kind ("pinned", "managed"; "system" = malloc, bookkeeping only) that are cached
    on free and reused for the next request of the same 512-B-rounded size."""

    def __init__(self, kind: str = "managed", limit_bytes: int = 0):
        self.kind = kind
        self.handle = ut_pool_create(UT_ALLOC[kind], limit_bytes)

    def alloc(self, nbytes: int) -> tuple[int, int]:
        return ut_pool_alloc(self.handle, nbytes)

    def free(self, host: int) -> None:
        ut_pool_free(self.handle, host)

    def release_cached(self) -> None:
        ut_pool_release_cached(self.handle)

    def stats(self) -> dict:
        return ut_pool_get_stats(self.handle)

    def table(self, rows: int, row_bytes: int, src=None) -> Table:
        return Table.from_pool(self, rows, row_bytes, src)

    def close(self) -> None:
        if getattr(self, "handle", None):
            ut_pool_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Coop:
    """One rank's side of a cooperative gather: the ranks of
    `group` (a torch.distributed process group, used only to move the IPC handles and, with
    sync="host", for the barriers between phases) gather their own index lists from `table`;
    rows requested by several ranks are fetched from host memory once, by their owner.

    sync="device": ut_coop_gather (phases ordered by flag words in peer memory, no host sync);
    sync="host": dispatch / fetch / combine with a stream sync and a group barrier between."""

    def __init__(self, table: Table, max_n: int, group=None, rank: int | None = None,
                 world: int | None = None, sync: str = "device", rows: int | None = None,
                 local: bool = False):
        """rows: None — `table` is the whole shared table; else the whole table's row count and
        `table` is this rank's partition (rows ut.Coop.partition_ids(rows, rb, world, rank)).
        local: every rank lives in THIS process (one host thread per GPU, each creating its rank
        with its device current); no process group is used — call `open_local` on every rank
        with all ranks' Coop objects before the first step (sync="device" only)."""
        import torch.distributed as dist
        if world is None:
            world = dist.get_world_size(group) if dist.is_initialized() else 1
        if rank is None:
            rank = dist.get_rank(group) if dist.is_initialized() else 0
        assert sync in ("device", "host")
        self.table, self.world, self.rank, self.sync, self.group = table, world, rank, sync, group
        self.max_n = int(max_n)
        self.rows = int(rows) if rows is not None else table.rows
        if rows is None:
            self.handle = ut_coop_create(table.handle, world, rank, self.max_n)
        else:
            self.handle = ut_coop_create_partitioned(table.handle, self.rows, world, rank, self.max_n)
        if local:
            assert sync == "device", "in-process ranks synchronise on the device"
        elif world > 1:
            # every rank must agree on the layout of the symmetric regions it is about to map
            mine = (ut_coop_export(self.handle),
                    (world, self.max_n, self.rows, table.row_bytes, rows is not None))
            allh = [None] * world
            dist.all_gather_object(allh, mine, group=group)
            shapes = {h[1] for h in allh}
            if len(shapes) != 1:
                self.close()
                raise UTError(UT_EINVAL, f"ranks disagree on (world, max_n, rows, row_bytes, partitioned): "
                                         f"{sorted(shapes)}")
            ut_coop_open(self.handle, b"".join(h[0] for h in allh))
            dist.barrier(group=group)

    def open_local(self, ranks: list["Coop"]) -> None:
        """Map the other in-process ranks' regions (ut_coop_open_local); this rank's device must
        be current."""
        ut_coop_open_local(self.handle, [r.handle for r in ranks])

    @staticmethod
    def partition_ids(rows: int, row_bytes: int, world: int, rank: int):
        return ut_coop_partition_ids(rows, row_bytes, world, rank)

    def _barrier(self, stream) -> None:
        import torch
        import torch.distributed as dist
        s = torch.cuda.current_stream() if stream is None else stream
        s.synchronize()
        if self.world > 1:
            dist.barrier(group=self.group)

    def gather(self, idx, out=None, stream=None):
        """out[i] = table row idx[i] (uint8 [n, row_bytes] CUDA tensor); every rank calls it."""
        import torch
        assert idx.is_cuda and idx.dtype == torch.int64 and idx.is_contiguous()
        n = idx.numel()
        rb = self.table.row_bytes
        if out is None:
            out = torch.empty((n, rb), dtype=torch.uint8, device=idx.device)
        else:
            assert out.is_cuda and out.is_contiguous() and out.numel() * out.element_size() >= n * rb
        sh = _stream_handle(stream)
        if self.sync == "device":
            ut_coop_gather(self.handle, idx.data_ptr(), n, out.data_ptr(), sh)
            return out
        ut_coop_dispatch(self.handle, idx.data_ptr(), n, sh)
        self._barrier(stream)
        ut_coop_fetch(self.handle, sh)
        self._barrier(stream)
        ut_coop_combine(self.handle, out.data_ptr(), sh)
        return out

    __getitem__ = gather

    def stats(self) -> dict:
        return ut_coop_get_stats(self.handle)

    def error_pos(self, stream=None) -> int:
        return ut_coop_error_pos(self.handle, _stream_handle(stream))

    def close(self) -> None:
        if getattr(self, "handle", None):
            ut_coop_release(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Graph:
    """A host-resident CSR graph sampled by GPU threads."""

    def __init__(self, indptr_addr: int, indices_addr: int, n_nodes: int, n_edges: int, keep=None):
        self._keep = keep
        self.n_nodes, self.n_edges = int(n_nodes), int(n_edges)
        self.handle = ut_graph_register(indptr_addr, indices_addr, n_nodes, n_edges)

    def set_option(self, option: str) -> None:
        ut_graph_set_option(self.handle, option)

    def sample(self, seeds, fanouts, seed: int, out=None, stream=None):
        """Minibatch node list (CUDA int64 tensor, seeds first) for CUDA int64 `seeds`."""
        import torch
        assert seeds.is_cuda and seeds.dtype == torch.int64 and seeds.is_contiguous()
        cap = seeds.numel()
        for f in fanouts:
            cap += cap * int(f)
        cap = min(cap, self.n_nodes)
        if out is None or out.numel() < cap:
            out = torch.empty(max(1, cap), dtype=torch.int64, device=seeds.device)
        n = ut_sample(self.handle, seeds.data_ptr(), seeds.numel(), list(fanouts), seed,
                      out.data_ptr(), out.numel(), _stream_handle(stream))
        return out[:n]

    def launches(self) -> int:
        return int(_lib.ut_graph_launches(self.handle))

    def capacity(self, n_seeds: int, fanouts) -> int:
        return ut_sample_capacity(n_seeds, list(fanouts), self.n_nodes)

    def sample_async(self, seeds, fanouts, seed: int, nodes, n_dev, stream=None) -> None:
        """Enqueue a sample into `nodes` (CUDA int64, >= capacity) and its count into `n_dev`
        (CUDA int64 [1]) with no host synchronisation (graph-capturable)."""
        ut_sample_async(self.handle, seeds.data_ptr(), seeds.numel(), list(fanouts), seed,
                        nodes.data_ptr(), nodes.numel(), n_dev.data_ptr(), _stream_handle(stream))

    def close(self) -> None:
        if getattr(self, "handle", None):
            ut_graph_release(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
