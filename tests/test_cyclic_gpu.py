"""The fused block-cyclic multi-GPU scan (ls_inclusive_scan_multi) on one
GPU: W virtual GPUs run concurrently as W cooperative kernels on W streams,
each on its own share of the SMs, exchanging stripe aggregates through each
other's exchange regions exactly as physical GPUs do through NVLink peer
memory.  The result, reassembled in block-cyclic order, must equal the
oracle scan of the global array."""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_1604_04815_b200 import _native as N
    from paper_1604_04815_b200 import scan as S
    from paper_1604_04815_b200.errors import raise_for_status
    return N, S, raise_for_status


class VirtualGPUs:
    """W virtual GPUs on one device: own exchange region, workspace and stream
    each; the peer table points at each other's regions."""

    def __init__(self, env, W, dtype, n, grid=None):
        N, S, raise_for_status = env
        self.L, self.S, self.raise_ = N.lib(), S, raise_for_status
        self.W, self.dtype, self.n = W, dtype, n
        self.dt = S.dtype_code(dtype)
        sms = S.query_config(dtype, n)["sms"]
        self.grid = grid or sms // W
        self.xbytes = self.L.ls_xchg_bytes(self.dt, W, n)
        self.regions, self.wss, self.streams = [], [], []
        for _ in range(W):
            p = ctypes.c_void_p()
            raise_for_status(self.L.ls_device_alloc(self.xbytes, ctypes.byref(p)))
            raise_for_status(self.L.ls_workspace_init(p.value, self.xbytes, None))
            self.regions.append(p.value)
            wb = self.L.ls_workspace_bytes(self.dt, n)
            w = torch.zeros(wb + 256, dtype=torch.uint8, device="cuda")
            off = (-w.data_ptr()) % 128
            self.wss.append((w, w.data_ptr() + off, wb))
            self.streams.append(torch.cuda.Stream())
        self.peers = torch.tensor(self.regions, dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()

    def __call__(self, x_parts, op="add", exclusive=False, carry=None, spin_budget=5_000_000):
        L, S = self.L, self.S
        outs = [torch.empty_like(xp) for xp in x_parts]
        tots = [torch.empty(1, dtype=self.dtype, device="cuda") for _ in range(self.W)]
        cin = None if carry is None else torch.tensor([carry], dtype=self.dtype, device="cuda")
        fn = L.ls_exclusive_scan_multi if exclusive else L.ls_inclusive_scan_multi
        torch.cuda.synchronize()
        # watchdog armed so that a protocol bug fails the test instead of hanging
        self.raise_(L.ls_debug_config(spin_budget, -1, 0))
        try:
            for r in range(self.W):
                rc = fn(S.op_code(op), self.dt, x_parts[r].data_ptr(), outs[r].data_ptr(), self.n,
                        None if cin is None else cin.data_ptr(), tots[r].data_ptr(), self.wss[r][1],
                        self.wss[r][2], r, self.W, self.regions[r], self.xbytes, self.peers.data_ptr(),
                        self.grid, self.streams[r].cuda_stream)
                self.raise_(rc)
            torch.cuda.synchronize()
        finally:
            L.ls_debug_config(0, -1, 0)
        for r in range(self.W):
            self.raise_(L.ls_workspace_error(self.wss[r][1], self.wss[r][2], self.streams[r].cuda_stream))
        return outs, tots

    def launch(self, x_parts, outs, n, op="add"):
        """Enqueue one call of n local elements per virtual GPU on its own
        stream, no synchronisation (the caller arms the watchdog and syncs)."""
        L, S = self.L, self.S
        for r in range(self.W):
            self.raise_(L.ls_inclusive_scan_multi(S.op_code(op), self.dt, x_parts[r].data_ptr(), outs[r].data_ptr(),
                                                  n, None, None, self.wss[r][1], self.wss[r][2], r, self.W,
                                                  self.regions[r], self.xbytes, self.peers.data_ptr(), self.grid,
                                                  self.streams[r].cuda_stream))

    def close(self):
        torch.cuda.synchronize()
        for p in self.regions:
            self.L.ls_device_free(p)


def run_virtual(env, x_parts, **kw):
    v = VirtualGPUs(env, len(x_parts), x_parts[0].dtype, x_parts[0].numel())
    try:
        outs, tots = v(x_parts, **kw)
    finally:
        v.close()
    return outs, tots, v.grid


def assemble(parts, stripe):
    """Block-cyclic local shares -> global order."""
    W = len(parts)
    n = parts[0].size
    k_full = n // stripe
    out = []
    for k in range(k_full):
        for g in range(W):
            out.append(parts[g][k * stripe:(k + 1) * stripe])
    if n % stripe:
        for g in range(W):
            out.append(parts[g][k_full * stripe:])
    return np.concatenate(out)


@pytest.mark.parametrize("tok,W", [("i32", 2), ("i64", 2), ("f32", 4), ("f64", 2), ("i32", 8), ("i64", 3)])
def test_virtual_gpus_match_global_scan(env, oracle_lib, tok, W):
    N, S, _ = env
    tdt = {"i32": torch.int32, "i64": torch.int64, "f32": torch.float32, "f64": torch.float64}[tok]
    tile = S.query_multi_config(tdt, 1 << 20)["tile_elems"]
    sms = S.query_config(tdt, 1 << 20)["sms"]
    grid = sms // W
    stripe = grid * tile
    n = 5 * stripe + 3 * tile + 123  # several full rounds and a short last one
    parts = [oracle_lib.generate_input(n, tok, [g, n, W]) for g in range(W)]
    xd = [torch.from_numpy(p).cuda() for p in parts]
    outs, tots, grid = run_virtual(env, xd)
    glob = assemble(parts, stripe)
    y = assemble([o.cpu().numpy() for o in outs], stripe)
    ref = oracle_lib.c_sequential_scan(glob)[0]
    if tok[0] == "i":
        assert np.array_equal(y, ref)
        assert all(t.item() == ref[-1] for t in tots)
    else:
        assert oracle_lib.validate_output(glob, y, ref=ref) is None
        # every GPU folds the same stripe totals in the same order
        assert len({t.cpu().numpy().tobytes() for t in tots}) == 1


@pytest.mark.parametrize("op", ["add", "max", "min"])
def test_virtual_gpus_ops_exclusive_carry(env, oracle_lib, op):
    N, S, _ = env
    W = 2
    tile = S.query_multi_config(torch.int64, 1 << 20)["tile_elems"]
    grid = S.query_config(torch.int64, 1 << 20)["sms"] // W
    stripe = grid * tile
    n = 3 * stripe + 77
    parts = [oracle_lib.generate_input(n, "i64", [g, 9]) for g in range(W)]
    xd = [torch.from_numpy(p).cuda() for p in parts]
    glob = assemble(parts, stripe)
    outs, _, _ = run_virtual(env, xd, op=op, exclusive=True)
    y = assemble([o.cpu().numpy() for o in outs], stripe)
    assert np.array_equal(y, oracle_lib.exclusive_scan(glob, op))
    if op == "add":
        outs, tots, _ = run_virtual(env, xd, carry=12345)
        y = assemble([o.cpu().numpy() for o in outs], stripe)
        ref, tot = oracle_lib.c_sequential_scan(glob, carry=np.int64(12345))
        assert np.array_equal(y, ref) and tots[0].item() == tot


def test_repeated_calls_alternate_parity(env, oracle_lib):
    # back-to-back calls on the same exchange regions (parity double buffer),
    # alternating operators: results stay exact
    N, S, _ = env
    W = 2
    tile = S.query_multi_config(torch.int32, 1 << 20)["tile_elems"]
    grid = S.query_config(torch.int32, 1 << 20)["sms"] // W
    n = 2 * grid * tile + 5
    parts = [oracle_lib.generate_input(n, "i32", [g, 1]) for g in range(W)]
    xd = [torch.from_numpy(p).cuda() for p in parts]
    glob = assemble(parts, grid * tile)
    v = VirtualGPUs(env, W, torch.int32, n, grid)
    try:
        for i in range(6):
            op = ("add", "max", "min")[i % 3]
            outs, _ = v(xd, op=op)
            assert np.array_equal(assemble([o.cpu().numpy() for o in outs], grid * tile),
                                  oracle_lib.sequential_scan(glob, op=op)), (i, op)
    finally:
        v.close()


@pytest.mark.slow
def test_two_pow_33_over_eight_virtual_gpus(env):
    # BASELINE configs[4]: 2^33 i32 over 8 GPUs, here 8 virtual GPUs of one
    # B200 (2^30 elements each, 64 GiB in + out), checked on the device with
    # the exact difference identity inside stripes and the stripe heads
    # against the block-cyclic prefix of the stripe sums
    N, S, _ = env
    W, n = 8, 1 << 30
    free, _ = torch.cuda.mem_get_info()
    if free < 72 * (1 << 30):
        pytest.skip("needs ~72 GiB of free device memory")
    g = torch.Generator(device="cuda").manual_seed(7)
    xs = [torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g) for _ in range(W)]
    v = VirtualGPUs(env, W, torch.int32, n)
    try:
        ys, tots = v(xs)
    finally:
        v.close()
    stripe = v.grid * S.query_multi_config(torch.int32, n)["tile_elems"]
    rounds = (n + stripe - 1) // stripe
    sums = torch.empty(rounds, W, dtype=torch.int64, device="cuda")
    for r in range(W):
        for k in range(rounds):
            sums[k, r] = xs[r][k * stripe:(k + 1) * stripe].sum(dtype=torch.int64)
    order = sums.reshape(-1).to(torch.int32).to(torch.int64)
    excl = (torch.cumsum(order, 0) - order).reshape(rounds, W).to(torch.int32)
    for r in range(W):
        x, y = xs[r], ys[r]
        for k in range(rounds):
            lo, hi = k * stripe, min(n, (k + 1) * stripe)
            assert torch.equal(y[lo + 1:hi] - y[lo:hi - 1], x[lo + 1:hi])
            assert y[lo] == (excl[k, r] + x[lo]).to(torch.int32)
    total = order.sum().to(torch.int32)
    assert all(t.item() == total.item() for t in tots)


def test_back_to_back_calls_of_unequal_length(env, oracle_lib):
    """consecutive calls with different n on the same exchange
    regions (a long call, a short one ending in a partial round, long again),
    enqueued back to back on every virtual GPU's own stream with no host
    synchronisation in between, so a fast GPU's next call overlaps a slow
    GPU's current one: the parity halves of the exchange region are laid out
    for the region's capacity, not the call's round count."""
    N, S, raise_ = env
    W = 3
    tile = S.query_multi_config(torch.int32, 1 << 20)["tile_elems"]
    # half the SMs per virtual GPU: each stream may hold its current call and
    # the next one (launched early through programmatic dependent launch), and
    # all of them must fit on the one device at once
    grid = S.query_config(torch.int32, 1 << 20)["sms"] // (2 * W)
    stripe = grid * tile
    n_big = 4 * stripe + 17
    lengths = [n_big, stripe + 3 * tile + 5, n_big, 2 * stripe, 3 * tile + 1, n_big]
    parts = [oracle_lib.generate_input(n_big, "i32", [g, 7]) for g in range(W)]
    xd = [torch.from_numpy(p).cuda() for p in parts]
    v = VirtualGPUs(env, W, torch.int32, n_big, grid)
    outs = [[torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(W)] for n in lengths]
    torch.cuda.synchronize()
    raise_(v.L.ls_debug_config(5_000_000, -1, 0))
    try:
        for i, n in enumerate(lengths):
            v.launch(xd, outs[i], n, op=("add", "max")[i % 2])
        torch.cuda.synchronize()
    finally:
        v.L.ls_debug_config(0, -1, 0)
    try:
        for r in range(W):
            raise_(v.L.ls_workspace_error(v.wss[r][1], v.wss[r][2], v.streams[r].cuda_stream))
        for i, n in enumerate(lengths):
            glob = assemble([p[:n] for p in parts], stripe)
            y = assemble([o.cpu().numpy() for o in outs[i]], stripe)
            assert np.array_equal(y, oracle_lib.sequential_scan(glob, op=("add", "max")[i % 2])), (i, n)
    finally:
        v.close()


@pytest.mark.parametrize("op", ["max", "min"])
@pytest.mark.parametrize("exclusive", [False, True])
def test_virtual_gpus_f64_maxmin_ties(env, op, exclusive):
    """The fused block-cyclic kernel's f64 max/min (transposed row scans,
    order-free reducers with the NaN screen) on data with signed zeros,
    NaN payloads and infinities: raw bits against numpy's sequential fold."""
    N, S, _ = env
    W = 2
    tile = S.query_multi_config(torch.float64, 1 << 20)["tile_elems"]
    grid = S.query_config(torch.float64, 1 << 20)["sms"] // W
    stripe = grid * tile
    n = 3 * stripe + 2 * tile + 45
    rng = np.random.default_rng([11, n])
    sign = -1.0 if op == "max" else 1.0
    parts = []
    for g in range(W):
        x = sign * rng.random(n)
        pos = rng.choice(n, size=40, replace=False)
        x[pos[:30]] = np.where(rng.random(30) < 0.5, -0.0, 0.0)
        x[pos[30:35]] = np.array([np.inf, -np.inf, 2.0 ** 1020, -(2.0 ** 1020), 0.0])
        if g == 1:  # NaNs with payloads late in the second GPU's data
            x[pos[35:]] = np.array([0x7FF8000000000123, 0xFFF800000000BEEF, 0x7FF8000000000000,
                                    0xFFF8000000000000, 0x7FF8000000000777], np.uint64).view(np.float64)
        parts.append(x)
    xd = [torch.from_numpy(p).cuda() for p in parts]
    outs, _, _ = run_virtual(env, xd, op=op, exclusive=exclusive)
    glob = assemble(parts, stripe)
    y = assemble([o.cpu().numpy() for o in outs], stripe)
    inc = (np.maximum if op == "max" else np.minimum).accumulate(glob)
    ref = np.concatenate([[-np.inf if op == "max" else np.inf], inc[:-1]]) if exclusive else inc
    bad = np.flatnonzero(y.view(np.uint64) != ref.view(np.uint64))
    assert bad.size == 0, f"{bad.size} mismatching bits, first at {bad[:5]}"
