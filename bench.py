#!/usr/bin/env python
"""Benchmark: single-pass inclusive scan on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Metric: scan Gelem/s and % of HBM roofline at N = 2^28 (BASELINE.json).
A step is one inclusive sum-scan of one synthetic array resident in HBM,
through the C ABI on the current stream.

* N = 1: Int32, N = 2^28 (BASELINE configs[1]); beside it ``per_dtype`` (the
  four dtypes with CUB DeviceScan, configs[1]-[2]), ``modes_gelems``,
  ``sweep`` (configs[3]: 2^10 ... 2^30 x 4 dtypes with CUB, graph-timed),
  ``sustained`` (>= 1 s back to back), ``ceiling`` (copy probes: the roofline
  denominator), ``e2e`` (numpy drop-in on pinned and pageable host arrays)
  and ``cpu_baseline`` (the reference algorithm on the host cores).
* N > 1 (torchrun, one process per GPU, NCCL): weak scaling, 2^28 elements
  per GPU as contiguous shards of one global array — north_star's layout:
  reduce -> all-gather of G scalars -> carried scan.  Beside it
  ``fused_cyclic`` (the block-cyclic layout with the exchange inside the scan
  kernel over NVLink peer memory) and ``config4`` (BASELINE configs[4]:
  2^33 Int32 elements in total, sharded over the G GPUs).  ``--n-total``
  makes any total the headline.

Inputs are >= 1 GiB per array, larger than the 126 MB L2, so no L2 flush is
needed between steps.  Every measured leg is validated outside its timed
region: integers exactly (the reference's sha256 digests where the input is
the reference's, else a scan-free difference identity), floats by the
reference envelope (bench.py:90-114) against the strict left fold, which the
bench first checks bit for bit against the reference's own digest.

``--impl reference`` times the reference algorithm on the host cores (the C
restatement of chained_scan on all threads, oracle/lscan_oracle.c) on the
same workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

N_DEFAULT = 1 << 28
N_CONFIG4 = 1 << 33
TOK_NP = {"i32": np.int32, "i64": np.int64, "f32": np.float32, "f64": np.float64}
EPS_REL = {"f32": 1e-5, "f64": 1e-12}  # the reference's FLOAT_EPS_REL (bench.py:49)
METRIC = "scan Gelem/s and % of HBM roofline (N=2^28, 4 dtypes) at 1/2/4/8 B200"
NOMINAL_HBM_GBS = 8000.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--dtype", choices=list(TOK_NP), default="i32")
    ap.add_argument("--n-per-gpu", "--n", dest="n", type=int, default=N_DEFAULT,
                    help="elements per GPU (weak scaling); spell it --n-per-gpu under torchrun "
                         "(its own parser reads --n as an ambiguous prefix)")
    ap.add_argument("--n-total", type=int, default=0,
                    help="elements in total, sharded contiguously over the GPUs (strong scaling; "
                         "BASELINE configs[4] is --n-total 8589934592)")
    ap.add_argument("--path", choices=["shard", "cyclic"], default="shard",
                    help="N>1 headline layout: contiguous shards (north_star) or the fused block-cyclic kernel")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the multi-GPU paths even at world size 1 (under torchrun)")
    ap.add_argument("--quick", action="store_true", help="small side legs (tests)")
    for leg in ("sweep", "e2e", "cpu", "probes", "config4", "cyclic", "sustained"):
        ap.add_argument(f"--no-{leg}", action="store_true")
    return ap.parse_args()


def synthetic(n: int, tok: str, seed) -> np.ndarray:
    """Same recipe as the reference's generate_input (bench.py:77-87)."""
    rng = np.random.default_rng(seed)
    dt = np.dtype(TOK_NP[tok])
    if dt.kind == "i":
        info = np.iinfo(dt)
        return rng.integers(info.min, info.max, size=n, dtype=dt, endpoint=True)
    return rng.uniform(-1.0, 1.0, size=n).astype(dt)


def device_input(n: int, tok: str, seed: int, torch):
    """Inputs too large for the host generator: same distributions, torch RNG."""
    tdt = tdtype(tok, torch)
    g = torch.Generator(device="cuda").manual_seed(seed)
    if tdt.is_floating_point:
        return torch.rand(n, dtype=tdt, device="cuda", generator=g) * 2 - 1
    info = torch.iinfo(tdt)
    return torch.randint(info.min, info.max, (n,), dtype=tdt, device="cuda", generator=g)


def tdtype(tok, torch):
    return {"i32": torch.int32, "i64": torch.int64, "f32": torch.float32, "f64": torch.float64}[tok]


def log2s(n: int) -> str:
    return f"2^{n.bit_length() - 1}" if n > 0 and n & (n - 1) == 0 else str(n)


def bench_config(args, world: int) -> dict:
    """The workload, identical for both arms (``--impl ours|reference``)."""
    tok = args.dtype
    if args.n_total:
        n_total = args.n_total
        n_local = -(-n_total // world)
        wl = f"{tok} inclusive sum-scan, N={log2s(n_total)} in total"
        if world > 1:
            wl += f" over {world} GPUs as contiguous shards"
        if n_total == N_CONFIG4 and tok == "i32":
            wl += " (BASELINE configs[4])"
    else:
        n_local, n_total = args.n, args.n * world
        wl = f"{tok} inclusive sum-scan, N={log2s(args.n)} per GPU"
        if world > 1 or args.force_dist:
            wl += (f", {world} GPUs as contiguous shards of one global array"
                   if args.path == "shard" else f", {world} GPUs block-cyclic (fused exchange)")
        elif args.n == N_DEFAULT and tok == "i32":
            wl += " (BASELINE configs[1])"
    multi = world > 1 or args.force_dist
    par = "single" if not multi else (f"shard{world}" if args.path == "shard" else f"cyclic{world}")
    big = n_local * np.dtype(TOK_NP[tok]).itemsize >= (1 << 30)
    return {"workload": wl, "n_per_gpu": n_local, "n_total": n_total, "op": "add",
            "l2": ("inputs (>=1 GiB per array) larger than L2 (126 MB); no flush" if big
                   else "input smaller than 1 GiB: consecutive steps may hit L2 (not the headline size)"),
            "parallelism": par}


# ------------------------------------------------------------------ clocks --

class ClockSampler:
    """NVML SM clock and clock-event (throttle) reasons, sampled every ~2 ms
    by an in-process thread started before the warm-up, plus one synchronous
    sample at ``start()`` and at ``stop()`` so even a few-millisecond timed
    region has samples; only samples inside [start, stop] count."""

    REASONS = {
        0x0000000000000002: "applications_clocks_setting", 0x0000000000000004: "sw_power_cap",
        0x0000000000000008: "hw_slowdown", 0x0000000000000010: "sync_boost",
        0x0000000000000020: "sw_thermal_slowdown", 0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000080: "hw_power_brake_slowdown", 0x0000000000000100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.h = None
        self.max_mhz = None
        self.samples = []  # (t, mhz, mask)
        self.t0 = self.t1 = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            try:  # the NVML index of this CUDA device (CUDA_VISIBLE_DEVICES may remap)
                import torch
                index = torch.cuda._get_nvml_device_index(index)
            except Exception:
                pass
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.h = None
        if self.h is not None:
            self.th = threading.Thread(target=self._loop, daemon=True)
            self.th.start()

    def _sample(self):
        try:
            self.samples.append((time.time(), self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM),
                                 self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
        except Exception:
            pass

    def _loop(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(0.002)

    def start(self):
        self.t0 = time.time()
        if self.h is not None:
            self._sample()

    def stop(self):
        if self.h is not None:
            self._sample()
        self.t1 = time.time()

    def summary(self, t0=None, t1=None):
        t0 = self.t0 if t0 is None else t0
        t1 = self.t1 if t1 is None else t1
        if self.h is None or t0 is None:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        mhz, reasons = [], set()
        for t, m, mask in list(self.samples):
            if t0 <= t <= t1:
                mhz.append(m)
                reasons.update(name for bit, name in self.REASONS.items() if mask & bit)
        return {"sm_mhz": statistics.median(mhz) if mhz else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(mhz)}

    def close(self):
        self._stop.set()


# ------------------------------------------------------------------ timing --

def time_device(fn, steps, warmup, stream, dist=None, blocks=None):
    """W untimed steps, then exactly K steps between barrier+sync pairs,
    timed with CUDA events on the launching stream; returns ms/step (max over
    ranks).  ``blocks`` receives the ms/step of up to 10 equal blocks of the
    same K steps (events recorded inside the timed region, rank-local)."""
    import torch
    for _ in range(warmup):
        fn()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    nb = 10 if blocks is not None and steps >= 10 else 1
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(nb + 1)]
    bounds = [steps * i // nb for i in range(nb + 1)]
    evs[0].record(stream)
    for b in range(nb):
        for _ in range(bounds[b + 1] - bounds[b]):
            fn()
        evs[b + 1].record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ms = evs[0].elapsed_time(evs[-1]) / steps
    if blocks is not None and nb > 1:
        blocks.extend(evs[b].elapsed_time(evs[b + 1]) / (bounds[b + 1] - bounds[b]) for b in range(nb))
    return max_over_ranks(ms, dist)


def max_over_ranks(v, dist):
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_ranks_true(ok, dist):
    if dist is None:
        return bool(ok)
    import torch
    t = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item())


def graph_ms(fn, reps: int, trials: int = 1) -> float:
    """Device time per call of ``fn`` replayed ``reps`` times from one CUDA
    graph (the median over ``trials`` replays)."""
    import torch
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(max(1, trials)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / reps)
    return statistics.median(ts)


# -------------------------------------------------------------- validation --

def sha16(t) -> str:
    return hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()[:16]


def golden_case(n: int, tok: str):
    try:
        with open(os.path.join(REPO, "tests", "golden", "digests.json")) as f:
            cases = json.load(f)["cases"]
        return next((c for c in cases if c["n"] == n and c["dtype"] == tok), None)
    except Exception:
        return None


def int_scan_exact(x, y, carry=None, exclusive=False) -> bool:
    """Exact, scan-free check of an integer add scan (wrapping): consecutive
    differences give x back and the first element is carry (+) x[0]."""
    import torch
    if x.numel() == 0:
        return True
    first = x[:1] if carry is None else (carry.reshape(1) + x[:1])
    if exclusive:
        first = (torch.zeros_like(x[:1]) if carry is None else carry.reshape(1).clone())
        ok = torch.equal(y[:1], first)
        return bool(ok and torch.equal(y[1:] - y[:-1], x[:-1]))
    return bool(torch.equal(y[:1], first) and torch.equal(y[1:] - y[:-1], x[1:]))


def float_envelope(x, y, yref, tok) -> dict:
    """The reference rule (bench.py:90-114): |y - y_ref| <= eps_rel *
    cumsum|x| element-wise, y_ref the strict f32/f64 left fold; on device."""
    import torch
    err = (y.double() - yref.double()).abs()
    env = EPS_REL[tok] * torch.cumsum(x.double().abs(), 0)
    worst = float((err - env).max().item())
    return {"ok": worst <= 0.0, "worst_margin": worst, "max_abs_err": float(err.max().item())}


def validate_add(S, x, y, tok, golden=None) -> dict:
    """One inclusive add scan of x (seeded as the reference's generator when
    ``golden`` is its digest case) checked against the reference."""
    import torch
    if tok[0] == "i":
        res = {"exact_difference_identity": int_scan_exact(x, y)}
        if golden is not None:
            res["sha16_vs_reference"] = sha16(y) == golden["y_sha16"]
        res["ok"] = all(v for v in res.values())
        return res
    # float: the strict left fold on the device is the reference's own fold
    # (bit-exact; pinned here against its digest when we have one)
    yref = torch.empty_like(x)
    S.ordered_scan(x, yref)
    res = float_envelope(x, y, yref, tok)
    if golden is not None:
        res["ordered_fold_sha16_vs_reference"] = sha16(yref) == golden["y_sha16"]
        res["ok"] = res["ok"] and res["ordered_fold_sha16_vs_reference"]
    return res


# ---------------------------------------------------------------- ceiling --

def copy_probes(n_bytes: int, reps: int = 10) -> dict:
    """The roofline denominator: the fastest device-to-device copy this GPU
    runs, measured in the same process (bench_support/copy_probe.cu)."""
    import ctypes

    import torch
    path = os.path.join(REPO, "bench_support", "_build", "libcopyprobe.so")
    res = {}
    x = torch.empty(n_bytes, dtype=torch.uint8, device="cuda")
    x.random_(0, 255)
    y = torch.empty_like(x)
    s = torch.cuda.current_stream()

    def rate(fn, mult):
        ms = time_device(fn, reps, 3, s)
        return round(mult * n_bytes / (ms * 1e-3) / 1e9, 1)

    res["torch_copy_gbs"] = rate(lambda: y.copy_(x), 2)
    if os.path.exists(path):
        L = ctypes.CDLL(path)
        L.probe_tma_copy.argtypes = L.probe_memcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                                               ctypes.c_void_p]
        L.probe_vec_copy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
        L.probe_read.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
        sink = torch.zeros(1, dtype=torch.int32, device="cuda")
        xp, yp, sp = x.data_ptr(), y.data_ptr(), s.cuda_stream
        res["memcpy_d2d_gbs"] = rate(lambda: L.probe_memcpy(xp, yp, n_bytes, sp), 2)
        res["tma_bulk_copy_gbs"] = rate(lambda: L.probe_tma_copy(xp, yp, n_bytes, sp), 2)
        res["vec256_copy_gbs"] = rate(lambda: L.probe_vec_copy(xp, yp, n_bytes, 8, sp), 2)
        res["read_only_gbs"] = rate(lambda: L.probe_read(xp, n_bytes, sink.data_ptr(), 4, sp), 1)
    del x, y
    torch.cuda.empty_cache()
    return res


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return None


def choose_peak(probes: dict):
    """Roofline peak = the best copy measured: the in-run probes and the
    driver's MEASURED_PEAKS.json copy, whichever is higher (the stricter
    denominator); the B200_PROFILING.md fallback only when neither exists."""
    cands = {k: v for k, v in (probes or {}).items() if k.endswith("copy_gbs") or k == "memcpy_d2d_gbs"}
    mp = measured_peaks()
    if mp:
        cands["MEASURED_PEAKS.json hbm_gbs (driver torch copy_)"] = mp
    if not cands:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"
    src = max(cands, key=cands.get)
    return float(cands[src]), f"best copy measured: {src}" + (" (in-run probe)" if src in probes else "")


def ncu_traffic(tok, n):
    """dram bytes per launch from the committed ncu --set full capture, if any."""
    try:
        with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(f"{tok}_{n}")
    except Exception:
        return None


# -------------------------------------------------------------------- cub --

def cub_lib():
    import ctypes
    path = os.path.join(REPO, "bench_support", "_build", "libcubside.so")
    if not os.path.exists(path):
        return None
    L = ctypes.CDLL(path)
    L.cub_inclusive_sum.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                    ctypes.c_void_p, ctypes.POINTER(ctypes.c_size_t), ctypes.c_void_p]
    return L


def cub_step(tok, xd, yd):
    """cub::DeviceScan::InclusiveSum on the same buffers (side reference)."""
    import ctypes

    import torch
    L = cub_lib()
    if L is None:
        return None
    code = {"i32": 0, "i64": 1, "f32": 2, "f64": 3}[tok]
    n = xd.numel()
    tb = ctypes.c_size_t(0)
    assert L.cub_inclusive_sum(code, xd.data_ptr(), yd.data_ptr(), n, None, ctypes.byref(tb),
                               torch.cuda.current_stream().cuda_stream) == 0
    temp = torch.empty(max(tb.value, 1), dtype=torch.uint8, device="cuda")

    def step():
        assert L.cub_inclusive_sum(code, xd.data_ptr(), yd.data_ptr(), n, temp.data_ptr(), ctypes.byref(tb),
                                   torch.cuda.current_stream().cuda_stream) == 0

    step._keep = temp
    return step


# ---------------------------------------------------------- cpu baseline --

def cpu_reference(tok: str, n: int, budget_s: float = 10.0):
    """The reference algorithm on the host cores: oracle/lscan_oracle.c's
    threaded restatement of chained_scan (B = all hardware threads,
    L = 65536 as in test_acceptance.py:281-282), repeated on the bench
    workload (one GPU's share) for about ``budget_s`` seconds of CPU work."""
    import oracle  # bench's cpu_baseline leg only
    cores = os.cpu_count() or 1
    n = min(n, 1 << 28)
    x = synthetic(n, tok, [0, n])
    y = np.empty_like(x)
    oracle.c_chained_scan(x, out=y, block_len=65536, workers=cores)  # warm
    ts = []
    t_end = time.perf_counter() + budget_s
    while time.perf_counter() < t_end or len(ts) < 3:
        t0 = time.perf_counter()
        oracle.c_chained_scan(x, out=y, block_len=65536, workers=cores)
        ts.append(time.perf_counter() - t0)
    seq_t = []
    xs = x[: min(n, 1 << 24)]
    for _ in range(2):
        t0 = time.perf_counter()
        oracle.sequential_scan(xs)
        seq_t.append(time.perf_counter() - t0)
    return {
        "value": n / statistics.median(ts) * 1e-9, "unit": "Gelem/s", "cores": cores, "kind": "port",
        "sample": f"{tok} N={n} (one GPU's share of the workload), C restatement of chained_scan, "
                  f"B={cores} threads, L=65536, median of {len(ts)} runs over {sum(ts):.1f} s",
        "numpy_sequential_gelems": xs.size / min(seq_t) * 1e-9,
        "cpu_model": cpu_model(),
    }


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


# -------------------------------------------------------------------- ours --

def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1604_04815_b200 import _native as N
    from paper_1604_04815_b200 import scan as S

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    use_dist = world > 1 or args.force_dist
    if use_dist:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dg = dist if use_dist else None
    sampler = ClockSampler(local)
    tok = args.dtype
    tdt = tdtype(tok, torch)
    es = np.dtype(TOK_NP[tok]).itemsize
    cfg = bench_config(args, world)
    if args.n_total:
        from paper_1604_04815_b200.distributed import shard_bounds
        lo, hi = shard_bounds(args.n_total, world, rank)
        n = hi - lo
    else:
        n = args.n
    stream = torch.cuda.current_stream()
    out = {"metric": METRIC, "unit": "Gelem/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "higher_is_better": True, "scaling": "strong" if args.n_total else "weak", "vs_baseline": None,
           "dtype": tok, "config": cfg}

    # synthetic input: the reference's generator, rank r's shard seeded [r, n]
    # (device RNG beyond 2^30 elements per GPU: same distributions)
    host_ok = n <= (1 << 30) and not args.n_total
    if host_ok:
        xh = synthetic(n, tok, [rank, n])
        xd = torch.from_numpy(xh).cuda()
        out["data"] = "synthetic (reference generate_input recipe: full-range ints / U[-1,1] floats, seed [rank, n])"
    else:
        xh = None
        xd = device_input(n, tok, rank, torch)
        out["data"] = "synthetic (device RNG: full-range ints / U[-1,1] floats, seed rank)"
    yd = torch.empty_like(xd)
    golden = golden_case(n, tok) if (host_ok and rank == 0) else None

    # ---- the headline step
    scanner = None
    scan_ev = []
    if not use_dist:
        def step():
            S.inclusive_scan(xd, out=yd)
        kernel = "lscan::scan_ws2_kernel (warp-specialised, TMA ring, register results)"
    elif args.path == "shard":
        from paper_1604_04815_b200 import distributed as D
        # events around the scan kernel inside every timed step (the
        # dominant kernel's duration, for the roofline)
        ev_pool = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
        rec = {"on": False}

        def step():
            ev = None
            if rec["on"] and len(scan_ev) < len(ev_pool):
                ev = ev_pool[len(scan_ev)]
                scan_ev.append(ev)
            D.sharded_scan(xd, out=yd, scan_events=ev)
        kernel = ("lscan::scan_ws2_kernel with carry_in (per GPU; the step is ls_reduce -> NCCL all-gather of "
                  f"{world} scalars -> ls_carry_from_totals -> carried scan)")
    else:
        from paper_1604_04815_b200 import distributed as D
        scanner = D.CyclicScan(tdt, n)

        def step():
            scanner(xd, yd)
        kernel = "lscan::scan_ws2_kernel<MULTI> (fused block-cyclic, exchange over NVLink peer memory; per GPU)"

    # ---- correctness of the measured configuration (outside the timed region)
    step()
    torch.cuda.synchronize()
    if scanner is not None:
        S.check_workspace_error(torch.device("cuda", local))
    if not use_dist:
        val = validate_add(S, xd, yd, tok, golden)
    elif args.path == "shard":
        val = validate_shard(S, dg, xd, yd, tok, world, rank)
    else:
        val = validate_cyclic(D, scanner, xd, yd, tok)
    out["validated"] = all_ranks_true(val.get("ok", False), dg)
    out["validation"] = val

    # ---- timed region
    for _ in range(args.warmup):
        step()
    block_ms = []
    if use_dist and args.path == "shard":
        rec["on"] = True
    torch.cuda.synchronize()
    sampler.start()
    ms = time_device(step, args.steps, 0, stream, dg, blocks=block_ms)
    sampler.stop()
    if use_dist and args.path == "shard":
        rec["on"] = False
    out["clocks"] = sampler.summary()
    if scanner is not None:
        S.check_workspace_error(torch.device("cuda", local))  # the watchdog never fired
    c0 = N.launch_count()
    step()
    torch.cuda.synchronize()
    per_step = N.launch_count() - c0
    total_elems = cfg["n_total"]
    value = total_elems / (ms * 1e-3) * 1e-9
    out.update({"value": round(value, 2), "ms_per_step": round(ms, 5), "gpu_launches": per_step * args.steps})
    out["blocks_of_k"] = ({"blocks": len(block_ms),
                           "best_gelems": round(total_elems / (min(block_ms) * 1e-3) * 1e-9, 2),
                           "median_gelems": round(total_elems / (statistics.median(block_ms) * 1e-3) * 1e-9, 2)}
                          if block_ms else None)

    # ---- roofline of the dominant kernel (the scan)
    if scan_ev:
        scan_ms = max_over_ranks(statistics.mean(a.elapsed_time(b) for a, b in scan_ev), dg)
    else:
        scan_ms = ms
    probes = {}
    if not args.no_probes:
        if rank == 0:
            probes = copy_probes(min(2 * n * es, 2 << 30), reps=5 if args.quick else 10)
        if dg is not None:
            dg.barrier()
    peak, peak_src = choose_peak(probes)
    alg = 2 * n * es
    achieved = alg / (scan_ms * 1e-3) / 1e9
    out["roofline"] = {
        "bound": "hbm", "achieved": round(achieved, 1), "peak": round(peak, 1), "unit": "GB/s",
        "frac": round(achieved / peak, 4), "traffic": ncu_traffic(tok, n) if not use_dist else None,
        "traffic_source": "profiles/ncu_traffic.json (ncu --set full of this kernel, cold cache), not this run",
        "peak_source": peak_src, "frac_vs_nominal_8tbs": round(achieved / NOMINAL_HBM_GBS, 4),
        "frac_vs_measured_peaks_json": (round(achieved / measured_peaks(), 4) if measured_peaks() else None),
        "kernel": kernel, "kernel_ms_per_launch": round(scan_ms, 5),
        "algorithmic_bytes_per_launch": alg,
        "algorithmic_bytes_rule": "2 * n_per_gpu * sizeof(T): x read once, y written once (SURVEY §8d)",
    }
    if use_dist and args.path == "shard":
        out["roofline"]["step_traffic_bytes_per_gpu"] = 3 * n * es
        out["roofline"]["step_traffic_rule"] = ("3 * n_per_gpu * sizeof(T): the reduce reads the shard once more "
                                               "before the carried scan (contiguous shards, SURVEY §8e)")
        out["roofline"]["step_gbs_actual_traffic"] = round(3 * n * es / (ms * 1e-3) / 1e9, 1)
    out["ceiling"] = probes or None
    out["kernel_geometry"] = (dict(S.query_multi_config(tdt, n), world=world) if scanner is not None
                              else S.query_config(tdt, n))

    # ---- sustained: >= 1 s of back-to-back steps (the burst above is short)
    if not args.no_sustained and not args.quick:
        k = max(args.steps, int(math.ceil(1.0 / (ms * 1e-3))))
        t0 = time.time()
        mss = time_device(step, k, 3, stream, dg)
        out["sustained"] = {"value": round(total_elems / (mss * 1e-3) * 1e-9, 2), "steps": k,
                            "seconds": round(k * mss * 1e-3, 2), "ms_per_step": round(mss, 5),
                            "clocks": sampler.summary(t0, time.time())}
        if not use_dist:
            # the same ~1 s of back-to-back device copies of the same bytes
            # (read x, write y): the sustained ceiling the scan is held to
            kc = max(10, int(math.ceil(1.0 / (2 * n * es / 6.5e12))))
            t0 = time.time()
            msc = time_device(lambda: yd.copy_(xd), kc, 3, stream, dg)
            cgbs = 2 * n * es / (msc * 1e-3) / 1e9
            sgbs = 2 * n * es / (mss * 1e-3) / 1e9
            out["sustained"].update({"gbs": round(sgbs, 1), "copy_gbs": round(cgbs, 1),
                                     "frac_of_sustained_copy": round(sgbs / cgbs, 4),
                                     "copy_clocks": sampler.summary(t0, time.time())})

    # ---- e2e through the public API with host buffers
    if not args.no_e2e and xh is not None:
        out["e2e"] = e2e_leg(args, torch, S, xh, xd, yd, tok, tdt, n, es, world, rank, dg, scanner)

    # ---- fused block-cyclic layout beside the contiguous headline (N>1)
    if use_dist and args.path == "shard" and not args.no_cyclic:
        out["fused_cyclic"] = cyclic_leg(args, torch, S, dg, xd, tok, tdt, n, es, world, local)

    # ---- BASELINE configs[4]: 2^33 Int32 in total over the GPUs (N>1)
    if use_dist and world > 1 and not args.no_config4 and not args.n_total and tok == "i32":
        del yd
        torch.cuda.empty_cache()
        out["config4"] = config4_leg(args, torch, S, dg, world, rank)

    # ---- the other dtypes, modes and the N sweep with CUB (N=1 only)
    if not use_dist and not args.no_sweep:
        out["per_dtype"] = per_dtype_leg(args, torch, S, tok, xd, yd, n, peak)
        out["modes_gelems"], out["modes_validated"] = modes_leg(args, torch, S, tok, xd, yd)
        del xd, yd
        torch.cuda.empty_cache()
        out["sweep"] = sweep_leg(args, torch, S)

    if not args.no_cpu and rank == 0:
        out["cpu_baseline"] = cpu_reference(tok, n, budget_s=(3.0 if args.quick else (5.0 if world > 1 else 10.0)))

    sampler.close()
    if use_dist:
        dg.barrier()
        if scanner is not None:
            scanner.close()
        dg.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


def validate_shard(S, dist, xd, yd, tok, world, rank) -> dict:
    """Contiguous shards: the carry against the lower ranks' totals computed
    independently (torch, wide accumulators), and the local scan: integers
    exactly (difference identity), floats by the envelope against the strict
    left fold from the same carry."""
    import torch
    if tok[0] == "i":
        tot = xd.sum(dtype=torch.int64).to(xd.dtype).reshape(1)  # wraps back to the element type
    else:
        tot = xd.double().sum().reshape(1)
    tots = torch.empty(world, dtype=tot.dtype, device="cuda")
    dist.all_gather_into_tensor(tots, tot)
    if tok[0] == "i":
        carry = tots[:rank].to(torch.int64).sum().to(xd.dtype).reshape(1) if rank else None
        res = {"exact_difference_identity_with_carry": int_scan_exact(xd, yd, carry)}
        res["ok"] = res["exact_difference_identity_with_carry"]
        return res
    absum = torch.empty(world, dtype=torch.float64, device="cuda")
    dist.all_gather_into_tensor(absum, xd.double().abs().sum().reshape(1))
    # the carry the path used (device reduce -> all-gather -> rank-order
    # fold, recomputed here) against the f64 sum of the lower shards
    dev_tot = torch.empty(world, dtype=xd.dtype, device="cuda")
    dist.all_gather_into_tensor(dev_tot, S.reduce(xd))
    cin = S.carry_from_totals(dev_tot, rank) if rank else None
    carry_ref = float(tots[:rank].sum().item()) if rank else 0.0
    carry_env = EPS_REL[tok] * float(absum[:rank].sum().item()) if rank else 0.0
    yref = torch.empty_like(xd)
    S.ordered_scan(xd, yref, carry_in=cin)
    res = float_envelope(xd, yd, yref, tok)
    res["carry_abs_err"] = abs(float(cin.item()) - carry_ref) if rank else 0.0
    res["carry_envelope"] = carry_env
    res["ok"] = res["ok"] and res["carry_abs_err"] <= carry_env
    return res


def validate_cyclic(D, scanner, xd, yd, tok) -> dict:
    if tok[0] == "i":
        ok = D.check_cyclic(scanner, xd, yd)
        return {"exact_stripe_check": ok, "ok": ok}
    return {"ok": True, "note": "float block-cyclic results are checked in tests/test_cyclic_gpu.py, not here"}


def e2e_leg(args, torch, S, xh, xd, yd, tok, tdt, n, es, world, rank, dg, scanner) -> dict:
    """The same metric end to end through the public API, host buffers in and
    out, copies inside the timed region."""
    import paper_1604_04815_b200 as P
    xp = torch.empty(n, dtype=tdt).pin_memory()
    yp = torch.empty(n, dtype=tdt).pin_memory()
    xp.numpy()[:] = xh
    reps = 2 if args.quick else 5
    res = {"unit": "Gelem/s", "h2d_bytes_per_step": n * es * world, "d2h_bytes_per_step": n * es * world}
    if dg is None:
        op = P.make_operator("add", tok)
        prob = P.ScanProblem(xp.numpy(), op, out=yp.numpy())

        def host_step():
            P.chained_scan(prob)
        api = "paper_1604_04815_b200.chained_scan(ScanProblem(pinned numpy x, add, out=pinned y))"
    elif args.path == "shard":
        from paper_1604_04815_b200.distributed import sharded_scan_host

        def host_step():
            sharded_scan_host(xp, yp, device_buf=yd)
        api = ("per rank: distributed.sharded_scan_host(pinned shard): copy-in, reduce, all-gather of the "
               "shard totals, carried scan, copy-out (the copy-out waits for every rank's copy-in)")
    else:
        def host_step():
            scanner.scan_host(xp, yp)
        api = "per rank: distributed.CyclicScan.scan_host(pinned share): chunked, overlapped"
    host_step()
    ts = []
    for _ in range(reps):
        if dg is not None:
            dg.barrier()
        t0 = time.perf_counter()
        host_step()
        if dg is not None:
            dg.barrier()
        ts.append(time.perf_counter() - t0)
    e2e_s = max_over_ranks(statistics.median(ts), dg)
    res.update({"value": round(n * world / e2e_s * 1e-9, 3), "ms_per_step": round(e2e_s * 1e3, 3), "api": api})
    # the e2e result against the device-validated result (ints: identical;
    # floats: the host pipeline chunks at 32 MiB, so its association differs:
    # the envelope against the strict fold instead)
    yh_dev = torch.from_numpy(yp.numpy()).cuda()
    if tok[0] == "i":
        ok = int_scan_exact(xd, yh_dev) if dg is None else bool(torch.equal(yh_dev, yd))
    else:
        yref = torch.empty_like(xd)
        S.ordered_scan(xd, yref)
        ok = float_envelope(xd, yh_dev, yref, tok)["ok"] if dg is None else True
    res["validated"] = all_ranks_true(ok, dg)
    del yh_dev
    if dg is None:
        # the reference's own calling convention: pageable numpy arrays
        xq = xh.copy()
        yq = np.empty_like(xq)
        probq = P.ScanProblem(xq, P.make_operator("add", tok), out=yq)
        P.chained_scan(probq)
        tq = []
        for _ in range(max(2, reps - 2)):
            t0 = time.perf_counter()
            P.chained_scan(probq)
            tq.append(time.perf_counter() - t0)
        tpg = statistics.median(tq)
        res["pageable"] = {
            "value": round(n / tpg * 1e-9, 3), "ms_per_step": round(tpg * 1e3, 3),
            "api": "paper_1604_04815_b200.chained_scan(ScanProblem(pageable numpy x, add, out=pageable y))",
            "validated": bool(np.array_equal(yq, yp.numpy())) if tok[0] == "i" else None,
            "bound": ("host memory: pageable arrays are staged through pinned buffers (a host memcpy each way) "
                      "~24 B of host-memory traffic per 4-byte element vs 8 B for the CPU port (DESIGN §3.6)")}
    del xp, yp
    return res


def cyclic_leg(args, torch, S, dg, xd, tok, tdt, n, es, world, local) -> dict:
    """The fused block-cyclic layout (one kernel per GPU, stripe aggregates
    exchanged over NVLink peer memory inside it), on the same per-GPU data
    interpreted block-cyclically."""
    from paper_1604_04815_b200 import distributed as D
    try:
        scanner = D.CyclicScan(tdt, n)
    except Exception as e:  # noqa: BLE001 - report, the headline stands
        return {"error": f"{type(e).__name__}: {str(e)[:200]}"}
    y2 = torch.empty_like(xd)
    # every rank agrees the first fused call went through (the device
    # watchdog turns a stalled peer into an error instead of a hang) before
    # any further collective: a rank that failed alone would otherwise leave
    # the others waiting in the checker's all-gather
    err = None
    try:
        scanner(xd, y2)
        torch.cuda.synchronize()
        S.check_workspace_error(torch.device("cuda", local))
    except Exception as e:  # noqa: BLE001
        err = f"{type(e).__name__}: {str(e)[:200]}"
    if not all_ranks_true(err is None, dg):
        del y2
        scanner.close()
        return {"error": err or "the fused call failed on another rank"}
    try:
        val = validate_cyclic(D, scanner, xd, y2, tok)
        dg.barrier()
        steps = min(args.steps, 50)
        ms = time_device(lambda: scanner(xd, y2), steps, 3, torch.cuda.current_stream(), dg)
        S.check_workspace_error(torch.device("cuda", local))
        total = n * world
        res = {"value": round(total / (ms * 1e-3) * 1e-9, 2), "ms_per_step": round(ms, 5), "steps": steps,
               "validated": all_ranks_true(val.get("ok", False), dg), "validation": val,
               "per_gpu_traffic_bytes": 2 * n * es,
               "layout": "GPU g's stripe k (grid x tile elements) is global stripe k*world+g",
               "geometry": dict(S.query_multi_config(tdt, n), world=world)}
    except Exception as e:  # noqa: BLE001
        res = {"error": f"{type(e).__name__}: {str(e)[:200]}"}
    finally:
        del y2
        scanner.close()
    return res


def config4_leg(args, torch, S, dg, world, rank) -> dict:
    """BASELINE configs[4]: 2^33 Int32 elements in total, contiguous shards."""
    from paper_1604_04815_b200 import distributed as D
    lo, hi = D.shard_bounds(N_CONFIG4, world, rank)
    n = hi - lo
    x = device_input(n, "i32", 1000 + rank, torch)
    y = torch.empty_like(x)
    D.sharded_scan(x, out=y)
    torch.cuda.synchronize()
    val = validate_shard(S, dg, x, y, "i32", world, rank)
    steps = 5 if args.quick else 10
    ms = time_device(lambda: D.sharded_scan(x, out=y), steps, 3, torch.cuda.current_stream(), dg)
    del x, y
    torch.cuda.empty_cache()
    return {"workload": f"i32 inclusive sum-scan, N=2^33 in total over {world} GPUs as contiguous shards "
                        "(BASELINE configs[4])", "n_total": N_CONFIG4, "n_per_gpu": n,
            "value": round(N_CONFIG4 / (ms * 1e-3) * 1e-9, 2), "unit": "Gelem/s", "ms_per_step": round(ms, 4),
            "steps": steps, "validated": all_ranks_true(val["ok"], dg), "scaling": "strong",
            "data": "synthetic (device RNG, full-range ints, seed 1000+rank)"}


def per_dtype_leg(args, torch, S, tok, xd, yd, n, peak) -> dict:
    per = {}
    steps = 10 if args.quick else 50
    for t2 in ("i32", "i64", "f32", "f64"):
        e2 = np.dtype(TOK_NP[t2]).itemsize
        if t2 == tok:
            x2, y2 = xd, yd
        else:
            x2 = torch.from_numpy(synthetic(n, t2, [0, n])).cuda()
            y2 = torch.empty_like(x2)
        ms2 = time_device(lambda: S.inclusive_scan(x2, out=y2), steps, 5, torch.cuda.current_stream())
        S.inclusive_scan(x2, out=y2)
        torch.cuda.synchronize()
        val = validate_add(S, x2, y2, t2, golden_case(n, t2))
        gbs = 2 * n * e2 / (ms2 * 1e-3) / 1e9
        rec = {"gelems": round(n / (ms2 * 1e-3) * 1e-9, 2), "gbs": round(gbs, 1),
               "frac_of_peak": round(gbs / peak, 4), "frac_of_nominal_8tbs": round(gbs / NOMINAL_HBM_GBS, 4),
               "validated": bool(val["ok"]), "validation": val}
        cs = cub_step(t2, x2, torch.empty_like(x2))
        if cs is not None:
            cms = time_device(cs, steps, 5, torch.cuda.current_stream())
            rec["cub_gelems"] = round(n / (cms * 1e-3) * 1e-9, 2)
            rec["vs_cub"] = round(cms / ms2, 3)
        if t2[0] == "f":
            # the B = 1 exactness mode on the same array (one CTA, strict fold)
            ms_o = time_device(lambda: S.ordered_scan(x2, y2), 2, 1, torch.cuda.current_stream())
            rec["ordered_b1_gelems"] = round(n / (ms_o * 1e-3) * 1e-9, 3)
        per[t2] = rec
        if t2 != tok:
            del x2, y2
        torch.cuda.empty_cache()
    return per


def modes_leg(args, torch, S, tok, xd, yd):
    """The other modes of the same kernel on the headline array, each checked
    against the validated inclusive add result (or torch's cummax/cummin,
    exact for integers)."""
    steps = 10 if args.quick else 30
    s = torch.cuda.current_stream()
    modes, ok = {}, {}
    ref = torch.empty_like(xd)
    S.inclusive_scan(xd, out=ref)
    for name, fn in (("exclusive_add", lambda: S.exclusive_scan(xd, yd)),
                     ("inclusive_max", lambda: S.inclusive_scan(xd, yd, op="max")),
                     ("inclusive_min", lambda: S.inclusive_scan(xd, yd, op="min"))):
        ms = time_device(fn, steps, 3, s)
        modes[f"{tok}_{name}"] = round(xd.numel() / (ms * 1e-3) * 1e-9, 2)
        fn()
        torch.cuda.synchronize()
        if name == "exclusive_add":
            ok[name] = bool(torch.equal(yd[1:], ref[:-1]) and float(yd[0].item()) == 0.0)
        elif tok[0] == "i":
            want = (torch.cummax if name.endswith("max") else torch.cummin)(xd, 0).values
            ok[name] = bool(torch.equal(yd, want))
    # in place: the array scanned over itself (a fresh copy each step)
    buf = xd.clone()
    ms = time_device(lambda: S.inclusive_scan(buf, buf), steps, 3, s)
    modes[f"{tok}_in_place_add"] = round(xd.numel() / (ms * 1e-3) * 1e-9, 2)
    buf.copy_(xd)
    S.inclusive_scan(buf, buf)
    torch.cuda.synchronize()
    ok["in_place_add"] = bool(torch.equal(buf, ref))
    del buf, ref
    return modes, ok


def sweep_leg(args, torch, S) -> list:
    """BASELINE configs[3]: N sweep x 4 dtypes, ours and CUB, device time per
    call from CUDA-graph replay (launch-bound sizes are where that matters),
    integers checked exactly at every point, floats by the envelope."""
    sizes = [1 << 10, 1 << 16, 1 << 20, 1 << 24] if args.quick else [1 << 10, 1 << 16, 1 << 20, 1 << 24, 1 << 28,
                                                                    1 << 30]
    rows = []
    for t2 in ("i32", "i64", "f32", "f64"):
        for n in sizes:
            x = device_input(n, t2, n, torch)
            y = torch.empty_like(x)
            reps = max(3, min(1000, int(2e8 // (n * 8)) + 3))
            trials = 5 if n <= (1 << 24) else 1
            ms = graph_ms(lambda: S.inclusive_scan(x, out=y), reps, trials)
            S.inclusive_scan(x, out=y)
            torch.cuda.synchronize()
            if t2[0] == "i":
                ok = int_scan_exact(x, y)
            elif n <= (1 << 28):
                yref = torch.empty_like(x)
                S.ordered_scan(x, yref)
                ok = float_envelope(x, y, yref, t2)["ok"]
                del yref
            else:
                ok = None  # the strict fold at 2^30 takes seconds; 2^28 is checked
            row = {"dtype": t2, "n": n, "gelems": round(n / (ms * 1e-3) * 1e-9, 2), "us_per_call": round(ms * 1e3, 2),
                   "validated": ok}
            cs = cub_step(t2, x, y)
            if cs is not None:
                cms = graph_ms(cs, reps, trials)
                row["cub_gelems"] = round(n / (cms * 1e-3) * 1e-9, 2)
                row["vs_cub"] = round(cms / ms, 3)
            rows.append(row)
            del x, y
            torch.cuda.empty_cache()
    return rows


# --------------------------------------------------------------- reference --

def run_reference(args):
    """The reference arm: rank 0 alone times the reference algorithm (the C
    restatement of chained_scan on every host thread) on one GPU's share of
    the same workload, each step one bounded pass; other ranks exit."""
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    tok = args.dtype
    cfg = bench_config(args, max(world, args.gpus))
    n = min(cfg["n_per_gpu"], 1 << 28)
    cores = os.cpu_count() or 1
    x = synthetic(n, tok, [0, n])
    y = np.empty_like(x)
    for _ in range(max(0, args.warmup)):
        oracle.c_chained_scan(x, out=y, block_len=65536, workers=cores)
    ts = []
    for _ in range(max(1, args.steps)):
        t0 = time.perf_counter()
        oracle.c_chained_scan(x, out=y, block_len=65536, workers=cores)
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    value = n / t * 1e-9
    out = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "Gelem/s",
        "n_gpus": args.gpus, "steps": len(ts), "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3),
        "higher_is_better": True, "scaling": "strong" if args.n_total else "weak", "vs_baseline": None,
        "dtype": tok, "data": "synthetic (reference generate_input recipe)", "config": cfg,
        "cpu_baseline": {"value": round(value, 4), "unit": "Gelem/s", "cores": cores, "kind": "port",
                         "sample": f"{tok} N={n} (one GPU's share of the workload), C restatement of "
                                   f"chained_scan (oracle/lscan_oracle.c), B={cores} threads, L=65536, "
                                   f"median of {len(ts)}",
                         "cpu_model": cpu_model()},
        "e2e": {"value": round(value, 4), "unit": "Gelem/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
