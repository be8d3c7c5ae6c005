"""The unified-tensor API: Table 3 placement rules pinned cell by cell against
the paper's table and SPEC's examples (CPU), and the API's behaviour on a B200 (GPU): bit-exact
to("unified") round trips, unified[gpu_idx] through ut_gather == oracle, hybrid elementwise ops
== the same op on CPU tensors, output kinds per Table 3, memAdvise error codes."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
from paper_2101_07956_b200 import unified as U   # noqa: E402

P = lambda prop=True: U.Operand("unified", propagated=prop)          # noqa: E731
CPU_T, CPU_S, GPU_T = U.Operand("cpu"), U.Operand("cpu", scalar=True), U.Operand("gpu")


@pytest.mark.parametrize("ops,want", [
    # Table 3, row x column
    ([P(True), CPU_T], ("GPU", "UnifiedNonPropagation")),                 # R1 C1
    ([P(False), CPU_T], ("CPU", "UnifiedNonPropagation")),                # R1 C2, none prefers prop
    ([P(False), P(True), CPU_T], ("GPU", "UnifiedNonPropagation")),       # R1 C2, one prefers prop
    ([P(True), GPU_T], ("GPU", "GPU")),                                   # R2 C1
    ([P(False), GPU_T], ("GPU", "UnifiedPropagation")),                   # R2 C2
    ([P(True), CPU_S], ("GPU", "GPU")),                                   # R3 C1 (scalar)
    ([P(True)], ("GPU", "GPU")),                                          # R3 C1 (no others)
    ([P(False)], ("CPU", "UnifiedNonPropagation")),                       # R3 C2, none prefers
    ([P(False), P(True), CPU_S], ("GPU", "UnifiedNonPropagation")),       # R3 C2, one prefers
    # SPEC.md:133-137 examples
    ([P(False), P(True), GPU_T], ("GPU", "UnifiedPropagation")),
    ([P(True), CPU_T, GPU_T], ("GPU", "UnifiedNonPropagation")),          # R1 wins over R2
])
def test_table3_cells(ops, want):
    assert U.resolve_placement(ops) == want


def test_exhaustive_against_six_cell_lookup():
    """Every mixture of <= 3 operands and every propagation assignment maps to one of the six
    cells (SPEC.md:158 'Exhaustive rule coverage')."""
    import itertools
    kinds = [P(True), P(False), CPU_T, CPU_S, GPU_T]
    cells = set()
    for k in (1, 2, 3):
        for ops in itertools.product(kinds, repeat=k):
            if not any(o.kind == "unified" for o in ops):
                with pytest.raises(ValueError):
                    U.resolve_placement(ops)
                continue
            row = ("R1" if any(o.kind == "cpu" and not o.scalar for o in ops)
                   else "R2" if any(o.kind == "gpu" for o in ops) else "R3")
            col = "C1" if all(o.propagated for o in ops if o.kind == "unified") else "C2"
            cells.add((row, col, U.resolve_placement(ops)))
    assert {(r, c) for r, c, _ in cells} == {(r, c) for r in ("R1", "R2", "R3") for c in ("C1", "C2")}


def test_non_unified_raise_runtime_error():
    t = torch.zeros(3)
    assert U.is_unified(t) is False
    with pytest.raises(RuntimeError):
        U.set_propagatedToCUDA(t, True)
    with pytest.raises(RuntimeError):
        U.memAdvise(t, "SetReadMostly", "cpu")


@pytest.mark.gpu
def test_to_unified_round_trip_and_flags():
    x = torch.randn(1000, 37)
    x.view(torch.int32)[5, 3] = 0x7FC00001          # a NaN payload: compare bits
    u = U.to_unified(x)
    assert U.is_unified(u) and u.is_unified and u.propagatedToCUDA
    assert u.cpu_view().view(torch.int32).equal(x.view(torch.int32))
    assert u.cuda_view().cpu().view(torch.int32).equal(x.view(torch.int32))
    g = U.to_unified(x.cuda(), propagatedToCUDA=False)
    assert g.cpu_view().view(torch.int32).equal(x.view(torch.int32)) and not g.propagatedToCUDA
    h = u.table.handle
    U.set_propagatedToCUDA(u, False)            # no allocation or copy
    assert u.table.handle == h and not u.propagatedToCUDA
    ones = U.unified(128, 1.0)                  # torch.ones(128, device="unified")
    assert ones.cpu_view().eq(1).all() and ones.shape == (128,)


@pytest.mark.gpu
def test_indexing_with_gpu_tensor_is_the_gather():
    import oracle
    x = torch.randn(5000, 100)
    u = U.to_unified(x)
    idx = torch.randint(0, 5000, (3000,), device="cuda")
    out = u[idx]                                        # Table 3 R2 C1: GPU output
    assert out.is_cuda and out.shape == (3000, 100)
    want, _ = oracle.gather(x.numpy().view(np.uint8).reshape(-1), 5000, 400, idx.cpu().numpy())
    assert out.cpu().numpy().tobytes() == want.tobytes()
    U.set_propagatedToCUDA(u, False)
    out2 = u[idx]                                       # R2 C2: unified propagation output
    assert U.is_unified(out2) and out2.propagatedToCUDA
    assert out2.numpy().tobytes() == want.tobytes()
    out3 = u[idx.cpu()]                                 # R1 C2: CPU compute, unified non-prop
    assert U.is_unified(out3) and not out3.propagatedToCUDA
    assert out3.numpy().tobytes() == want.tobytes()


@pytest.mark.gpu
def test_hybrid_elementwise_ops_follow_table3():
    a = torch.arange(12, dtype=torch.float32).reshape(3, 4)
    b = torch.full((3, 4), 2.0)
    u = U.to_unified(a)                                  # propagated
    r = u + b                                            # R1 C1 -> GPU compute, unified non-prop
    assert U.is_unified(r) and not r.propagatedToCUDA and r.cpu_view().equal(a + b)
    r = u * b.cuda()                                     # R2 C1 -> GPU output
    assert r.is_cuda and r.cpu().equal(a * b)
    r = u - 1.5                                          # R3 C1 -> GPU output
    assert r.is_cuda and r.cpu().equal(a - 1.5)
    v = U.to_unified(a, propagatedToCUDA=False)
    r = v < 5.0                                          # R3 C2, none prefers -> CPU, unified
    assert U.is_unified(r) and r.cpu_view().equal(a < 5.0)
    r = v + b.cuda()                                     # R2 C2 -> unified propagation
    assert U.is_unified(r) and r.propagatedToCUDA and r.cpu_view().equal(a + b)
    r = u / v                                            # R3 C2, one prefers -> GPU, unified
    assert U.is_unified(r) and not r.propagatedToCUDA
    np.testing.assert_array_equal(r.numpy(), (a / a).numpy())


@pytest.mark.gpu
def test_mem_advise_returns_cuda_error_codes():
    x = torch.randn(256, 16)
    u = U.to_unified(x, advise="SetPreferredLocation", adviseDevice="cpu")
    assert u.advise_record[2] == 0                       # applied right after allocation
    assert U.memAdvise(u, "SetAccessedBy", "cuda:0") == 0
    assert U.memAdvise(u, "SetReadMostly", "cpu") == 0
    assert U.memAdvise(u, "UnsetReadMostly", "cpu") == 0
    p = U.to_unified(x, kind="pinned")
    assert U.memAdvise(p, "SetReadMostly", "cpu") != 0   # not managed memory: the runtime's code
    assert p.cpu_view().equal(x)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["managed", "pinned"])
def test_unified_tensors_recycle_their_blocks(kind):
    """a closed unified tensor's block serves the next tensor of the same rounded size
    with no new backend allocation; contents are the new tensor's, bit-exact."""
    x = torch.randn(1000, 25)                            # 100 000 B -> 100 352-B block
    u = U.to_unified(x, kind=kind)
    addr = u.table.host_addr
    before = U.allocator_stats(kind)
    u.close()
    y = torch.randn(1000, 25)
    v = U.to_unified(y, kind=kind)
    after = U.allocator_stats(kind)
    assert v.table.host_addr == addr
    assert after["backend_calls"] == before["backend_calls"]
    assert after["recycled_hits"] == before["recycled_hits"] + 1
    assert v.cpu_view().equal(y) and v.cuda_view().cpu().equal(y)
    idx = torch.tensor([999, 0, 17, 17], device="cuda")
    assert v[idx].cpu().equal(y[idx.cpu()])              # gathered from the recycled block
    w = U.to_unified(torch.randn(10, 25), kind=kind)     # another size: a fresh block
    assert U.allocator_stats(kind)["backend_calls"] == after["backend_calls"] + 1
    v.close()
    w.close()
    U.empty_cache()
    st = U.allocator_stats(kind)
    assert st["blocks_cached"] == 0 and st["bytes_cached"] == 0


@pytest.mark.gpu
def test_advised_block_is_restored_before_reuse():
    x = torch.randn(64, 64)
    u = U.to_unified(x, advise="SetReadMostly", adviseDevice="cpu")
    addr = u.table.host_addr
    u.close()                                            # advice restored, block cached
    v = U.to_unified(x)
    assert v.table.host_addr == addr and v.cpu_view().equal(x)
    assert v[torch.arange(64, device="cuda")].cpu().equal(x)
    v.close()
