"""Unified tensors: the paper's user-facing API over the library.

PyTorch-Direct adds a tensor kind that lives in host memory and that both CPU and GPU code
dereference (§4.1), with the APIs of Table 1 and Table 2
 and the placement rules of Table 3 (§4.3). This module provides them on
top of the C ABI, without a PyTorch fork:

* ``to_unified(t, propagatedToCUDA=True, advise=None, adviseDevice="cpu")`` — ``t.to("unified")``
  (a new library-owned allocation, ``ut_create``; the advice is applied right after allocation
  and before the data is copied in, as P:446-450 requires); ``unified(shape, fill, dtype)`` —
  ``torch.ones(128, device="unified")``.
* ``UnifiedTensor.is_unified``, ``set_propagatedToCUDA`` (flag only: no allocation or copy,
  P:434-435), ``memAdvise`` (cudaMemAdvise, returns the error code). The module-level
  ``is_unified`` / ``set_propagatedToCUDA`` / ``memAdvise`` accept any tensor and raise
  ``RuntimeError`` for non-unified ones.
* ``resolve_placement(operands)`` — Table 3, the six cells.
* Storage from the recycling unified allocator (§4.4; ``ut_pool_*``): a closed
  tensor's block serves the next tensor of the same rounded size; ``allocator_stats()``,
  ``empty_cache()``.
* ``u[idx]`` — ``unified_tensor[gpu_tensor]``: the rows are gathered by ``ut_gather``
  (the hot path) straight out of host memory; output GPU or unified per Table 3.
* Elementwise ``+ - * / < > <= >= ==`` with CPU tensors, GPU tensors, scalars and other unified
  tensors, computed where Table 3 says: on the GPU through a zero-copy CUDA view of the host
  memory (``__cuda_array_interface__`` on the mapped address), or on the CPU through a numpy
  view; unified outputs are new unified tensors written in place by the op.
"""
from __future__ import annotations

import operator
from dataclasses import dataclass

import numpy as np

from . import Pool, Table, UTError, ut_mem_advise

_ADVICE = {"SetPreferredLocation": 0, "UnsetPreferredLocation": 1, "SetAccessedBy": 2,
           "UnsetAccessedBy": 3, "SetReadMostly": 4, "UnsetReadMostly": 5}

# ---- the unified allocator (§4.4) ---------------------------------------------
# Every unified tensor's storage comes from one recycling pool per allocation kind: closing a
# tensor caches its block, and the next tensor of the same 512-B-rounded size reuses it without a
# cudaMallocManaged / cudaMemAdvise (or cudaHostAlloc) call — "adapts the allocation recycling
# mechanism from the PyTorch CUDA allocator to reduce the number of CUDA API invocations".
_POOLED = ("managed", "pinned")
_pools: dict = {}


def _pool(kind: str) -> Pool:
    if kind not in _pools:
        _pools[kind] = Pool(kind)
    return _pools[kind]


def allocator_stats(kind: str = "managed") -> dict:
    """Counters of the unified allocator for ``kind`` (backend calls, recycled hits, bytes)."""
    return _pool(kind).stats()


def empty_cache() -> None:
    """Return every cached unified block to CUDA (``torch.cuda.empty_cache`` for unified)."""
    for p in _pools.values():
        p.release_cached()


# ---- Table 3 -------------------------------------------------------------------------------------
GPU, CPU = "GPU", "CPU"
OUT_GPU, OUT_UNIFIED_PROP, OUT_UNIFIED_NONPROP = "GPU", "UnifiedPropagation", "UnifiedNonPropagation"


@dataclass(frozen=True)
class Operand:
    """What Table 3 needs to know about an operand."""
    kind: str                 # "unified" | "cpu" | "gpu"
    scalar: bool = False      # a CPU scalar (Python number or 0-d CPU tensor)
    propagated: bool = True   # unified only: propagatedToCUDA


def resolve_placement(operands) -> tuple[str, str]:
    """(compute device, output kind) for an operator with at least one unified operand, exactly
    as PAPER.md Table 3 lists the six cells:

    rows    R1 at least one operand is a non-scalar CPU tensor;
            R2 R1 does not apply and at least one operand is a GPU tensor;
            R3 all non-unified operands are CPU scalars, or there are none;
    columns C1 all unified operands prefer propagation; C2 at least one prefers non-propagation.
    """
    ops = list(operands)
    uni = [o for o in ops if o.kind == "unified"]
    if not uni:
        raise ValueError("no unified operand: Table 3 does not apply (use native dispatch)")
    all_prop = all(o.propagated for o in uni)
    any_prop = any(o.propagated for o in uni)
    if any(o.kind == "cpu" and not o.scalar for o in ops):                       # R1
        return (GPU if all_prop or any_prop else CPU), OUT_UNIFIED_NONPROP
    if any(o.kind == "gpu" for o in ops):                                        # R2
        return GPU, (OUT_GPU if all_prop else OUT_UNIFIED_PROP)
    # R3
    if all_prop:
        return GPU, OUT_GPU
    return (GPU if any_prop else CPU), OUT_UNIFIED_NONPROP


# ---- the tensor kind -------------------------------------------------------------------------
class _CudaArray:
    """__cuda_array_interface__ over a device address (zero-copy CUDA view for torch)."""

    def __init__(self, addr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(int(x) for x in shape), "typestr": typestr,
                                         "data": (int(addr), False), "version": 3, "strides": None}


class UnifiedTensor:
    """A dense tensor whose storage is a library-owned host allocation the GPU maps."""

    def __init__(self, shape, dtype, kind: str = "managed", propagatedToCUDA: bool = True,
                 advise: str | None = None, adviseDevice="cpu"):
        import torch
        self.shape = tuple(int(x) for x in shape)
        self.dtype = dtype
        self.kind = kind
        self.advise_record = None
        esize = torch.empty((), dtype=dtype).element_size()
        if len(self.shape) >= 2:      # rows = first dimension, as the paper's feature table
            rows, per_row = self.shape[0], int(np.prod(self.shape[1:]))
        else:                         # 1-D (or 0-d): one element per row
            rows, per_row = int(np.prod(self.shape)), 1
        rows = max(1, rows)
        self.row_bytes = max(1, per_row * esize)
        if kind in _POOLED:          # the recycling unified allocator (ut_pool_*)
            self.table = Table.from_pool(_pool(kind), rows, self.row_bytes)
        else:
            self.table = Table.create(rows, self.row_bytes, kind)
        self.propagatedToCUDA = bool(propagatedToCUDA)
        self.advise_record = None
        if advise is not None:                      # right after allocation
            self.memAdvise(advise, adviseDevice)

    # -- Table 1 / Table 2 -------------------------------------------------------------------
    @property
    def is_unified(self) -> bool:
        return True

    def set_propagatedToCUDA(self, value: bool) -> None:
        """Switch the placement hint: no allocation, deallocation or copy."""
        self.propagatedToCUDA = bool(value)

    def memAdvise(self, advise: str, adviseDevice="cpu") -> int:
        """cudaMemAdvise on the storage; returns the CUDA error code (Table 2)."""
        if advise not in _ADVICE:
            raise ValueError(f"unknown advise {advise!r}")
        dev = _device_index(adviseDevice)
        rc = ut_mem_advise(self.table.handle, _ADVICE[advise], dev)
        self.advise_record = (advise, adviseDevice, rc)
        return rc

    # -- views -------------------------------------------------------------------------------
    def _typestr(self) -> str:
        import torch
        return {torch.float32: "<f4", torch.float64: "<f8", torch.float16: "<f2",
                torch.int64: "<i8", torch.int32: "<i4", torch.int16: "<i2", torch.int8: "|i1",
                torch.uint8: "|u1", torch.bool: "|b1"}[self.dtype]

    def cpu_view(self):
        """torch CPU tensor aliasing the host storage (the CPU dereferences it directly)."""
        import torch
        n = int(np.prod(self.shape)) if self.shape else 1
        raw = self.table.array()
        esize = torch.empty((), dtype=self.dtype).element_size()
        return torch.from_numpy(raw[: n * esize]).view(self.dtype).reshape(self.shape)

    def cuda_view(self):
        """torch CUDA tensor aliasing the same host storage: GPU kernels read it over the link
        ("GPU kernels ... can directly access features since it can access unified tensor",
        P:331-332)."""
        import torch
        return torch.as_tensor(_CudaArray(self.table.host_addr, self.shape, self._typestr()),
                               device="cuda")

    def numpy(self):
        return self.cpu_view().numpy()

    # -- indexing: unified_tensor[gpu_tensor] (Table 1) -------------------------------
    def __getitem__(self, idx):
        import torch
        if not isinstance(idx, torch.Tensor) or idx.dtype not in (torch.int64, torch.int32) or idx.dim() != 1:
            raise TypeError("a unified tensor is indexed by a 1-D integer index tensor")
        op_idx = Operand("gpu") if idx.is_cuda else Operand("cpu", scalar=False)
        compute, out_kind = resolve_placement([Operand("unified", propagated=self.propagatedToCUDA), op_idx])
        n = idx.numel()
        out_shape = (n,) + self.shape[1:]
        if compute == CPU:
            src = self.cpu_view()
            res = src[idx.cpu().long()]
            return _place(res, out_kind, self.dtype)
        idx_d = idx.to(device="cuda", dtype=torch.int64).contiguous()
        if out_kind == OUT_GPU:
            out = torch.empty(out_shape, dtype=self.dtype, device="cuda")
            self.table.gather(idx_d, out=out.view(torch.uint8).view(-1))
            return out
        res = UnifiedTensor(out_shape, self.dtype, "managed",
                            propagatedToCUDA=(out_kind == OUT_UNIFIED_PROP))
        # the kernel stores the rows straight into the new unified tensor's mapped storage
        self.table.gather(idx_d, out=res.cuda_view().view(torch.uint8).view(-1))
        torch.cuda.current_stream().synchronize()
        return res

    # -- elementwise (Table 1 "unified_tensor + cpu_tensor", Table 3 placement) ---------------
    def _binary(self, other, fn, reverse=False):
        import torch
        ops = [self, other]
        desc = [_operand(x) for x in ops]
        compute, out_kind = resolve_placement(desc)
        args = [_as_compute(x, compute) for x in ops]
        if reverse:
            args.reverse()
        if out_kind == OUT_GPU:
            return fn(*args)
        res_t = fn(*args)                              # compute where Table 3 says
        res = UnifiedTensor(tuple(res_t.shape), res_t.dtype, "managed",
                            propagatedToCUDA=(out_kind == OUT_UNIFIED_PROP))
        dst = res.cuda_view() if compute == GPU else res.cpu_view()
        dst.copy_(res_t)
        if compute == GPU:
            torch.cuda.current_stream().synchronize()
        return res

    def __add__(self, o): return self._binary(o, operator.add)
    def __radd__(self, o): return self._binary(o, operator.add, reverse=True)
    def __sub__(self, o): return self._binary(o, operator.sub)
    def __rsub__(self, o): return self._binary(o, operator.sub, reverse=True)
    def __mul__(self, o): return self._binary(o, operator.mul)
    def __rmul__(self, o): return self._binary(o, operator.mul, reverse=True)
    def __truediv__(self, o): return self._binary(o, operator.truediv)
    def __lt__(self, o): return self._binary(o, operator.lt)
    def __le__(self, o): return self._binary(o, operator.le)
    def __gt__(self, o): return self._binary(o, operator.gt)
    def __ge__(self, o): return self._binary(o, operator.ge)
    def __eq__(self, o): return self._binary(o, operator.eq)
    __hash__ = object.__hash__

    def close(self) -> None:
        if getattr(self, "table", None) is None or not self.table.handle:
            return
        if self.advise_record is not None and self.kind == "managed":
            # the block goes back to the pool: restore the advice a fresh block has (Table 2)
            dev = self.table.info()["device"]
            for adv, where in (("UnsetReadMostly", "cpu"), ("SetPreferredLocation", "cpu"),
                               ("SetAccessedBy", dev)):
                ut_mem_advise(self.table.handle, _ADVICE[adv], _device_index(where))
        self.table.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __repr__(self):
        return (f"UnifiedTensor(shape={self.shape}, dtype={self.dtype}, "
                f"propagatedToCUDA={self.propagatedToCUDA})")


def _device_index(d) -> int:
    if isinstance(d, int):
        return d
    s = str(d)
    if s == "cpu":
        return -1
    if s.startswith("cuda"):
        return int(s.split(":")[1]) if ":" in s else 0
    raise ValueError(f"unknown device {d!r}")


def _operand(x) -> Operand:
    import torch
    if isinstance(x, UnifiedTensor):
        return Operand("unified", propagated=x.propagatedToCUDA)
    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            return Operand("gpu")
        return Operand("cpu", scalar=(x.dim() == 0))
    if isinstance(x, (int, float, bool)):
        return Operand("cpu", scalar=True)
    raise TypeError(type(x))


def _as_compute(x, compute):
    import torch
    if isinstance(x, UnifiedTensor):
        return x.cuda_view() if compute == GPU else x.cpu_view()
    if isinstance(x, torch.Tensor) and x.dim() > 0:
        return x.cuda() if compute == GPU else x.cpu()
    return x


def _place(res, out_kind, dtype):
    if out_kind == OUT_GPU:
        return res.cuda()
    u = UnifiedTensor(tuple(res.shape), res.dtype, "managed",
                      propagatedToCUDA=(out_kind == OUT_UNIFIED_PROP))
    u.cpu_view().copy_(res)
    return u


# ---- creation (Table 1 / Table 2) --------------------------------------------------------------
def to_unified(t, propagatedToCUDA: bool = True, advise: str | None = None, adviseDevice="cpu",
               kind: str = "managed") -> UnifiedTensor:
    """``t.to("unified")``: a unified copy of a CPU or GPU tensor, bit-equal contents."""
    import torch
    src = t.detach().contiguous()
    u = UnifiedTensor(tuple(src.shape), src.dtype, kind, propagatedToCUDA, advise, adviseDevice)
    if src.is_cuda:
        u.cuda_view().copy_(src)
        torch.cuda.current_stream().synchronize()
    else:
        u.cpu_view().copy_(src)
    return u


def unified(shape, fill=0, dtype=None, propagatedToCUDA: bool = True, **kw) -> UnifiedTensor:
    """``torch.ones(128, device="unified")`` and friends: a filled unified tensor."""
    import torch
    u = UnifiedTensor(tuple(shape) if not isinstance(shape, int) else (shape,),
                      dtype or torch.float32, kw.pop("kind", "managed"), propagatedToCUDA, **kw)
    u.cpu_view().fill_(fill)
    return u


def is_unified(t) -> bool:
    """Table 1 ``one_tensor.is_unified``."""
    return isinstance(t, UnifiedTensor)


def set_propagatedToCUDA(t, value: bool) -> None:
    """Table 2; a non-unified tensor raises RuntimeError."""
    if not isinstance(t, UnifiedTensor):
        raise RuntimeError("set_propagatedToCUDA: the tensor is not a unified tensor")
    t.set_propagatedToCUDA(value)


def memAdvise(t, advise: str, adviseDevice="cpu") -> int:
    """Table 2; a non-unified tensor raises RuntimeError."""
    if not isinstance(t, UnifiedTensor):
        raise RuntimeError("memAdvise: the tensor is not a unified tensor")
    return t.memAdvise(advise, adviseDevice)


__all__ = ["UnifiedTensor", "Operand", "resolve_placement", "to_unified", "unified", "is_unified",
           "allocator_stats", "empty_cache",
           "set_propagatedToCUDA", "memAdvise", "GPU", "CPU", "OUT_GPU", "OUT_UNIFIED_PROP",
           "OUT_UNIFIED_NONPROP", "UTError"]
