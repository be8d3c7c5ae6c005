"""Seeded synthetic inputs for the unified-tensor gather: host tables and index lists.

This module holds none of the gather's arithmetic. It is the one place both sides of a parity
check take their inputs from: the oracle (``oracle/``) and the CUDA path
(``paper_2101_07956_b200``) never import each other, only this.

* ``fill_table`` writes the self-identifying table content (``gen.c`` header).
* ``uniform_idx`` draws uniform-with-replacement row ids (the paper's microbenchmark "uses a
  random number generator (RNG) to generate random indices").
* ``HostBuffer`` owns plain host memory (anonymous mmap, optional guard pages, or a shared
  ``/dev/shm`` file for multi-process runs); registration/pinning is the library's job.
* ``graphsage`` builds GraphSAGE-shaped minibatch index lists.
"""
from __future__ import annotations

import ctypes
import mmap
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_SO = os.path.join(_HERE, "libutgen.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile gen.c into workloads/libutgen.so (gcc, OpenMP)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.run(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-Wall", "-o", tmp, _SRC, "-lm"],
                       check=True)
        os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.gen_splitmix64.restype = ctypes.c_uint64
        L.gen_splitmix64.argtypes = [ctypes.c_uint64]
        L.gen_fill_table.restype = None
        L.gen_fill_table.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                     ctypes.c_uint64, ctypes.c_int]
        L.gen_fill_table_on.restype = ctypes.c_int
        L.gen_fill_table_on.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                        ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int]
        L.gen_fill_rows.restype = None
        L.gen_fill_rows.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                    ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int]
        L.gen_uniform_idx.restype = None
        L.gen_uniform_idx.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                      ctypes.c_uint64]
        L.gen_chunglu_indptr.restype = ctypes.c_int64
        L.gen_chunglu_indptr.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_double, ctypes.c_uint64]
        L.gen_chunglu_indices.restype = None
        L.gen_chunglu_indices.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                          ctypes.c_double, ctypes.c_uint64, ctypes.c_int]
        L.gen_numa_nodes.restype = ctypes.c_int
        L.gen_numa_nodes.argtypes = []
        L.gen_bind_node.restype = ctypes.c_int
        L.gen_bind_node.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int]
        L.gen_interleave.restype = ctypes.c_int
        L.gen_interleave.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
        L.gen_map.restype = ctypes.c_void_p
        L.gen_map.argtypes = [ctypes.c_uint64, ctypes.c_int]
        L.gen_unmap.restype = ctypes.c_int
        L.gen_unmap.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
        L.gen_map_guarded.restype = ctypes.c_void_p
        L.gen_map_guarded.argtypes = [ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p),
                                      ctypes.POINTER(ctypes.c_uint64)]
        _lib = L
    return _lib


def splitmix64(x: int) -> int:
    return int(lib().gen_splitmix64(x & 0xFFFFFFFFFFFFFFFF))


def _addr(a) -> int:
    if isinstance(a, int):
        return a
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    raise TypeError(type(a))


def fill_table(dst, rows: int, rb: int, seed: int, threads: int = 0) -> None:
    """Write the self-identifying content of a rows x rb table at ``dst`` (array or address)."""
    if isinstance(dst, np.ndarray):
        assert dst.nbytes >= rows * rb
    lib().gen_fill_table(_addr(dst), rows, rb, seed & 0xFFFFFFFFFFFFFFFF, threads)


def fill_table_on(dst, rows: int, rb: int, seed: int, cpus: list[int]) -> bool:
    """fill_table's content written by one thread pinned to each CPU in ``cpus`` (first touch on
    their NUMA node). True when every thread ran pinned."""
    c = np.ascontiguousarray(cpus, dtype=np.int32)
    return lib().gen_fill_table_on(_addr(dst), rows, rb, seed & 0xFFFFFFFFFFFFFFFF,
                                   c.ctypes.data, int(c.size)) == 0


def fill_rows(dst, ids: np.ndarray, rb: int, seed: int, threads: int = 0) -> None:
    """Row k of ``dst`` = the content fill_table gives row ids[k] (zero row for ids[k] < 0): a
    partition or sub-table of chosen rows — table input, never an expected gather result."""
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    if isinstance(dst, np.ndarray):
        assert dst.nbytes >= ids.size * rb
    if ids.size:
        lib().gen_fill_rows(_addr(dst), ids.ctypes.data, ids.size, rb, seed & 0xFFFFFFFFFFFFFFFF, threads)


def uniform_idx(n: int, rows: int, seed: int) -> np.ndarray:
    """n row ids uniform with replacement over [0, rows) (int64)."""
    out = np.empty(n, dtype=np.int64)
    if n:
        lib().gen_uniform_idx(out.ctypes.data, n, rows, seed & 0xFFFFFFFFFFFFFFFF)
    return out


def numa_nodes() -> int:
    return int(lib().gen_numa_nodes())


def interleave(addr: int, nbytes: int) -> int:
    """Interleave the pages of [addr, addr+nbytes) over all NUMA nodes before first touch.
    Returns the node count used (0: single node, nothing to do; -1: mbind failed)."""
    return int(lib().gen_interleave(addr, nbytes))


def bind_node(addr: int, nbytes: int, node: int) -> bool:
    """Bind the pages of [addr, addr+nbytes) to one NUMA node before first touch."""
    return int(lib().gen_bind_node(addr, nbytes, node)) == 0


def gpu_numa_node(device_index: int = 0) -> int:
    """NUMA node of a CUDA device from sysfs (-1 when unknown)."""
    try:
        import torch
        p = torch.cuda.get_device_properties(device_index)
        path = f"/sys/bus/pci/devices/{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0/numa_node"
        return int(open(path).read().strip())
    except Exception:
        return -1


def node_cpus(node: int) -> list[int]:
    cpus = []
    try:
        for part in open(f"/sys/devices/system/node/node{node}/cpulist").read().strip().split(","):
            a, _, b = part.partition("-")
            cpus.extend(range(int(a), int(b or a) + 1))
    except OSError:
        pass
    return cpus


def decode_row_ids(rows_bytes: np.ndarray, rb: int) -> np.ndarray:
    """Row id encoded in the first min(rb, 8) bytes of each row of a self-identifying table.

    For rb < 8 only the low 8*rb bits of the id survive; callers compare modulo 2**(8*rb)."""
    a = np.asarray(rows_bytes, dtype=np.uint8).reshape(-1, rb)
    k = min(rb, 8)
    pad = np.zeros((a.shape[0], 8), dtype=np.uint8)
    pad[:, :k] = a[:, :k]
    return pad.view("<u8").reshape(-1).astype(np.int64)


class HostBuffer:
    """Plain (unpinned) host memory holding a table, placed at a chosen alignment.

    kind="anon":    anonymous mmap (THP-advised); the table starts ``offset`` bytes into it.
    kind="guarded": PROT_NONE pages on both sides and the table's last byte is the last byte
                    before the trailing guard page, so any over-read faults.
    kind="shm":     a MAP_SHARED ``/dev/shm`` file (``name``) that several processes map;
                    ``create`` decides who sizes it.
    """

    def __init__(self, nbytes: int, kind: str = "anon", offset: int = 0, hugepage: bool = True,
                 name: str | None = None, create: bool = True):
        self.nbytes = int(nbytes)
        self.kind = kind
        self._mm = None
        self._fd = None
        self._map_base = None
        self._map_len = 0
        self.path = None
        if kind == "anon":
            self._map_len = self.nbytes + offset + 4096
            base = lib().gen_map(self._map_len, 1 if hugepage else 0)
            if not base:
                raise MemoryError(f"mmap of {self._map_len} bytes failed")
            self._map_base = base
            self.addr = base + offset
        elif kind == "guarded":
            mb = ctypes.c_void_p()
            ml = ctypes.c_uint64()
            p = lib().gen_map_guarded(self.nbytes, ctypes.byref(mb), ctypes.byref(ml))
            if not p:
                raise MemoryError("guarded mmap failed")
            self._map_base = mb.value
            self._map_len = ml.value
            self.addr = p
        elif kind == "shm":
            assert name, "shm buffers need a name"
            self.path = os.path.join("/dev/shm", name)
            flags = os.O_RDWR | (os.O_CREAT if create else 0)
            self._fd = os.open(self.path, flags, 0o600)
            length = self.nbytes + offset
            if create:
                os.ftruncate(self._fd, length)
            self._mm = mmap.mmap(self._fd, length, mmap.MAP_SHARED,
                                 mmap.PROT_READ | mmap.PROT_WRITE)
            base = ctypes.addressof(ctypes.c_char.from_buffer(self._mm))
            self.addr = base + offset
        else:
            raise ValueError(kind)

    def array(self) -> np.ndarray:
        """uint8 numpy view of the table bytes (no copy)."""
        buf = (ctypes.c_uint8 * self.nbytes).from_address(self.addr)
        return np.ctypeslib.as_array(buf)

    def close(self, unlink: bool = False) -> None:
        if self._map_base is not None:
            lib().gen_unmap(self._map_base, self._map_len)
            self._map_base = None
        if self._mm is not None:
            try:
                self._mm.close()
            except BufferError:
                pass  # a numpy view is still alive; the mapping goes with the process
            self._mm = None
        if self._fd is not None:
            os.close(self._fd)
            self._fd = None
        if unlink and self.path and os.path.exists(self.path):
            os.unlink(self.path)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class CSRGraph:
    """An explicit host CSR graph (indptr int64[N+1], indices int32[E]) in plain host memory:
    the input of GPU-side neighbour sampling. Chung-Lu power law, see gen.c."""

    def __init__(self, n_nodes: int, n_edges: int, seed: int = 1, gamma: float = 2.5,
                 threads: int = 0):
        self.n_nodes = int(n_nodes)
        self._ip = HostBuffer((self.n_nodes + 1) * 8)
        self.indptr = np.ctypeslib.as_array(
            (ctypes.c_int64 * (self.n_nodes + 1)).from_address(self._ip.addr))
        self.n_edges = int(lib().gen_chunglu_indptr(self._ip.addr, self.n_nodes, n_edges, gamma, seed))
        self._ix = HostBuffer(max(1, self.n_edges) * 4)
        self.indices = np.ctypeslib.as_array(
            (ctypes.c_int32 * max(1, self.n_edges)).from_address(self._ix.addr))[: self.n_edges]
        lib().gen_chunglu_indices(self._ip.addr, self._ix.addr, self.n_nodes, gamma, seed, threads)

    @property
    def indptr_addr(self) -> int:
        return self._ip.addr

    @property
    def indices_addr(self) -> int:
        return self._ix.addr

    def close(self):
        self.indptr = self.indices = None
        self._ip.close()
        self._ix.close()
