"""pool_model — TEST INFRASTRUCTURE ONLY: the unified allocator's block recycling, replayed.

PAPER.md §4.4: "A new memory allocator is implemented to govern the memory allocation
for all unified tensors. It adapts the allocation recycling mechanism from the PyTorch CUDA
allocator to reduce the number of CUDA API invocations." The paper gives no parameters; this
model takes SPEC.md's reading (module unified-allocator) step by step, with the two
gaps it leaves filled as DESIGN.md reading R19 states:

* sizes are rounded up to a multiple of 512 B; a request of 0 B is a zero-capacity
  sentinel with no backend call, freeing it is a no-op;
* a cached block is reused only for a request of the same rounded size ("the same
  size-bucket", whole-block reuse, no splitting or coalescing); among several cached
  blocks of that size the most recently freed one is reused (R19: the paper's PyTorch allocator
  keeps its free blocks in a size-ordered set and SPEC only asks for best fit, which every block
  of one bucket is equally; last-in-first-out is the choice that makes "free(b); allocate(same
  size) -> b", hold);
* free returns a block to the cache, never to the backend; freeing a block that is not
  live is an error;
* a capacity limit bounds the bytes the backend holds (live + cached). When a fresh
  backend allocation would pass it, every cached block is returned to the backend first (R19:
  what the PyTorch CUDA allocator does before it reports out of memory) and the allocation is
  retried once; if it still does not fit, the request fails with out-of-memory and nothing changes
  but the emptied cache;
* release_cached() returns every cached block to the backend.

Only ``tests/`` import this module; the library's allocator (``csrc/ut_pool.cu``) shares nothing
with it. Pinned by tests/test_pool_model.py (SPEC's worked examples and closed forms: with no
limit, backend calls per size = that size's peak number of live blocks).
"""
from __future__ import annotations

GRANULE = 512


class PoolError(Exception):
    """An operation the allocator refuses: ``kind`` is "oom" or "invalid"."""

    def __init__(self, kind: str):
        super().__init__(kind)
        self.kind = kind


def round_up(nbytes: int) -> int:
    """Capacity of a request: the next multiple of 512 B; 0 stays 0."""
    return -(-nbytes // GRANULE) * GRANULE


class PoolModel:
    """Replay model. Blocks are named by integers in the order the backend creates them."""

    def __init__(self, limit: int = 0):
        self.limit = limit                # 0 = none
        self.live = {}                    # block id -> capacity
        self.cached = {}                  # capacity -> [block ids], most recently freed last
        self.held = 0                     # backend bytes: live + cached
        self.next_id = 1                  # 0 is the zero-capacity sentinel
        self.backend_calls = 0
        self.backend_frees = 0
        self.recycled_hits = 0

    # -- S:193-199 -----------------------------------------------------------------------------
    def allocate(self, nbytes: int) -> tuple[int, int]:
        """Returns (block id, capacity)."""
        if nbytes < 0:
            raise PoolError("invalid")
        cap = round_up(nbytes)
        if cap == 0:
            return 0, 0
        stack = self.cached.get(cap)
        if stack:                                        # same bucket cached: reuse, no backend call
            b = stack.pop()
            self.live[b] = cap
            self.recycled_hits += 1
            return b, cap
        if self.limit and self.held + cap > self.limit:  # would pass the limit: empty the cache
            self.release_cached()
            if self.held + cap > self.limit:
                raise PoolError("oom")
        b = self.next_id
        self.next_id += 1
        self.backend_calls += 1
        self.held += cap
        self.live[b] = cap
        return b, cap

    # -- S:200-208 -----------------------------------------------------------------------------
    def free(self, b: int) -> None:
        if b == 0:
            return
        if b not in self.live:
            raise PoolError("invalid")
        cap = self.live.pop(b)
        self.cached.setdefault(cap, []).append(b)

    def release_cached(self) -> None:
        for cap, stack in self.cached.items():
            self.backend_frees += len(stack)
            self.held -= cap * len(stack)
        self.cached = {}

    # -- S:209-214 -----------------------------------------------------------------------------
    def stats(self) -> dict:
        return {"backend_calls": self.backend_calls, "backend_frees": self.backend_frees,
                "recycled_hits": self.recycled_hits,
                "bytes_live": sum(self.live.values()),
                "bytes_cached": sum(c * len(s) for c, s in self.cached.items()),
                "blocks_live": len(self.live),
                "blocks_cached": sum(len(s) for s in self.cached.values())}


class NaiveModel:
    """The no-recycling allocator SPEC compares against: every non-empty request is a
    backend call, every free a backend free."""

    def __init__(self):
        self.backend_calls = 0
        self.live = {}
        self.next_id = 1

    def allocate(self, nbytes: int) -> tuple[int, int]:
        cap = round_up(nbytes)
        if cap == 0:
            return 0, 0
        b = self.next_id
        self.next_id += 1
        self.backend_calls += 1
        self.live[b] = cap
        return b, cap

    def free(self, b: int) -> None:
        if b:
            del self.live[b]
