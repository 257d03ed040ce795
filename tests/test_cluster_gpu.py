"""The latency kernel (small and mid n; lscan_cluster.cuh) against the
oracle: every dtype x operator x mode, sizes around its block tiles, its
one-cluster / several-cluster boundaries and its upper limit,
element-misaligned x and y, carry-in / total-out, in place.

Integers and max/min: bit-exact (also against the persistent kernel forced
on the same input).  Float add: the reference envelope
FLOAT_EPS_REL * cumsum|x| (bench.py:49, :90-114) and bit-reproducible.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOKS = ["i32", "i64", "f32", "f64"]
TDT = {"i32": torch.int32, "i64": torch.int64, "f32": torch.float32, "f64": torch.float64}


@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_1604_04815_b200 import scan
    return scan


def ref_scan(oracle_lib, x, op, exclusive):
    return oracle_lib.exclusive_scan(x, op) if exclusive else oracle_lib.sequential_scan(x, op=op)


def check(oracle_lib, x, y, op, exclusive, what):
    msg = oracle_lib.validate_output(x, y, exclusive=exclusive, op=op)
    assert msg is None, f"{what}: {msg}"


def sizes(S, tok):
    c = S.query_cluster(TDT[tok])
    B, one, top, Bm = c["block_elems"], c["one_cluster_elems"], c["max_elems"], c["mid_block_elems"]
    Cm = c["max_blocks"] * Bm  # one cluster of mid tiles
    mid = c["mid_max_elems"]    # beyond: large tiles
    return sorted({1, 2, 3, 5, 31, 32, 33, 1000, 1024, 4097, B - 1, B, B + 1, 2 * B + 7, 5 * B - 3,
                   one - 1, one, one + 1, Cm - 1, Cm, Cm + 1, 2 * Cm + Bm + 3, mid - 1, mid, mid + 1,
                   top - 3 * B + 1, top - 1, top})


def test_cluster_geometry(S):
    for tok in TOKS:
        c = S.query_cluster(TDT[tok])
        assert c["max_blocks"] in (8, 16), c
        es = 4 if tok in ("i32", "f32") else 8
        assert c["block_elems"] * es == 16384 and c["mid_block_elems"] * es == 32768
        assert c["capacity"] >= 1 and c["max_elems"] >= c["one_cluster_elems"]


@pytest.mark.parametrize("tok", TOKS)
@pytest.mark.parametrize("op", ["add", "max", "min"])
def test_cluster_kernel_parity(S, oracle_lib, tok, op):
    with S.force_path("cluster"):
        for n in sizes(S, tok):
            x = oracle_lib.generate_input(n, tok, [n, 3])
            xd = torch.from_numpy(x).cuda()
            for excl in (False, True):
                fn = S.exclusive_scan if excl else S.inclusive_scan
                y = fn(xd, op=op).cpu().numpy()
                check(oracle_lib, x, y, op, excl, f"{tok} {op} excl={excl} n={n}")


@pytest.mark.parametrize("tok", TOKS)
@pytest.mark.parametrize("which", ["one_cluster_elems", "mid_max_elems", "max_elems"])
def test_cluster_matches_persistent_kernel(S, oracle_lib, tok, which):
    """Same input through both kernels: ints and max/min bit-identical."""
    n = S.query_cluster(TDT[tok])[which] - 12345
    x = oracle_lib.generate_input(n, tok, [9, n])
    xd = torch.from_numpy(x).cuda()
    ops = ["add", "max", "min"] if tok[0] == "i" else ["max", "min"]
    for op in ops:
        with S.force_path("cluster"):
            a = S.inclusive_scan(xd, op=op).cpu().numpy()
        with S.force_path("persistent"):
            b = S.inclusive_scan(xd, op=op).cpu().numpy()
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), (tok, op)


@pytest.mark.parametrize("tok", TOKS)
@pytest.mark.parametrize("shift_x,shift_y", [(1, 0), (0, 1), (1, 1), (3, 2)])
def test_cluster_misaligned(S, oracle_lib, tok, shift_x, shift_y):
    with S.force_path("cluster"):
        for n in (7, 5000, S.query_cluster(TDT[tok])["max_elems"] - 3):
            x = oracle_lib.generate_input(n + shift_x, tok, [shift_x, n])
            xd = torch.from_numpy(x).cuda()[shift_x:]
            yd = torch.empty(n + shift_y, dtype=xd.dtype, device="cuda")[shift_y:]
            S.inclusive_scan(xd, out=yd)
            check(oracle_lib, x[shift_x:].copy(), yd.cpu().numpy(), "add", False, f"{tok} n={n} misaligned")


@pytest.mark.parametrize("tok", TOKS)
def test_cluster_carry_total_in_place(S, oracle_lib, tok):
    with S.force_path("cluster"):
        n = 150_001 if tok in ("i32", "f32") else 70_001
        x = oracle_lib.generate_input(n, tok, [4, n])
        cut = 40_000
        xd = torch.from_numpy(x).cuda()
        t1 = torch.empty(1, dtype=xd.dtype, device="cuda")
        t2 = torch.empty(1, dtype=xd.dtype, device="cuda")
        a = xd[:cut].clone()
        b = xd[cut:].clone()
        S.inclusive_scan(a, out=a, total_out=t1)  # in place
        S.inclusive_scan(b, out=b, carry_in=t1, total_out=t2)
        y = torch.cat([a, b]).cpu().numpy()
        check(oracle_lib, x, y, "add", False, f"{tok} carry chain")
        ref = oracle_lib.sequential_scan(x)
        if tok[0] == "i":
            assert t2.item() == ref[-1]
        else:
            assert abs(t2.item() - float(ref[-1])) <= 1e-5 * np.abs(x, dtype=np.float64).sum()
        # exclusive with a carry: y[0] = carry
        c = torch.from_numpy(x[:1].copy()).cuda()
        ye = S.exclusive_scan(xd[1:], carry_in=c).cpu().numpy()
        check(oracle_lib, x, np.concatenate([[0], ye]).astype(x.dtype), "add", True, f"{tok} excl carry")


def test_cluster_float_determinism(S, oracle_lib):
    with S.force_path("cluster"):
        for tok in ("f32", "f64"):
            n = S.query_cluster(TDT[tok])["max_elems"] - 1
            xd = torch.from_numpy(oracle_lib.generate_input(n, tok, [1, n])).cuda()
            ys = [S.inclusive_scan(xd).cpu().numpy() for _ in range(3)]
            for y in ys[1:]:
                assert np.array_equal(ys[0].view(np.uint8), y.view(np.uint8))


def test_auto_boundary(S, oracle_lib):
    """Either side of the cluster kernel's limit under the automatic choice."""
    for tok in TOKS:
        top = S.query_cluster(TDT[tok])["max_elems"]
        for n in (top, top + 1):
            x = oracle_lib.generate_input(n, tok, [2, n])
            y = S.inclusive_scan(torch.from_numpy(x).cuda()).cpu().numpy()
            check(oracle_lib, x, y, "add", False, f"{tok} n={n}")


def test_graph_capture_replay(S, oracle_lib):
    """Small scans captured in a CUDA graph replay correctly (no workspace state)."""
    x = oracle_lib.generate_input(40_000, "i32", [5, 5])
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        S.inclusive_scan(xd, out=yd)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            S.inclusive_scan(xd, out=yd)
    torch.cuda.synchronize()
    for seed in range(3):
        x2 = oracle_lib.generate_input(40_000, "i32", [seed, 6])
        xd.copy_(torch.from_numpy(x2))
        yd.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(yd.cpu().numpy(), oracle_lib.sequential_scan(x2))


@pytest.mark.parametrize("graph", [False, True])
@pytest.mark.parametrize("n", [30_001, 3_000_017])
def test_dependent_chain(S, oracle_lib, graph, n):
    """Back-to-back scans where each reads the previous one's output (the
    programmatic-dependent-launch overlap must keep the data dependency),
    with a torch kernel in between every few calls; eager and graph-replayed;
    on the latency kernel (30 001) and the persistent kernel (3 000 017)."""
    x0 = oracle_lib.generate_input(n, "i32", [8, 8])
    bufs = [torch.from_numpy(x0).cuda()] + [torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(12)]

    def chain():
        for i in range(12):
            S.inclusive_scan(bufs[i], out=bufs[i + 1])
            if i % 4 == 3:
                bufs[i + 1].add_(1)

    if graph:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            chain()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                chain()
        torch.cuda.synchronize()
        for b in bufs[1:]:
            b.zero_()
        g.replay()
    else:
        chain()
    torch.cuda.synchronize()
    want = x0
    with np.errstate(over="ignore"):
        for i in range(12):
            want = oracle_lib.sequential_scan(want)
            if i % 4 == 3:
                want = (want + np.int32(1)).astype(np.int32)
    assert np.array_equal(bufs[-1].cpu().numpy(), want)
