"""The C-ABI library loads and exports every symbol include/lscan.h declares;
host-side argument checks and the Python surface behave like the reference.
No compute calls: CPU only."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_1604_04815_b200 as P
from paper_1604_04815_b200 import _native as N
from paper_1604_04815_b200.distributed import shard_bounds

HEADER = os.path.join(N.INCLUDE, "lscan.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ls_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    names = declared_functions()
    assert len(names) >= 14
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(names) == sorted(N.EXPORTED)


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump -lelf {N.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def test_status_strings():
    assert N.status_string(0) == "LS_OK"
    assert N.status_string(N.LS_ERR_LIVENESS) == "LS_ERR_LIVENESS"
    assert N.status_string(N.LS_ERR_PROTOCOL) == "LS_ERR_PROTOCOL"
    assert N.lib().ls_abi_version() == 1


def test_workspace_bytes():
    lib = N.lib()
    # 32 KiB tiles: 8192 i32 / 4096 i64 elements; 8 / 16 bytes per slot, two slot arrays
    b32 = lib.ls_workspace_bytes(N.LS_I32, 1 << 28)
    b64 = lib.ls_workspace_bytes(N.LS_I64, 1 << 28)
    assert b32 >= 2 * (1 << 15) * 8 and b64 >= 2 * (1 << 16) * 16
    assert b32 % 256 == 0
    assert lib.ls_workspace_bytes(9, 10) == 0
    assert lib.ls_workspace_bytes(N.LS_I32, -1) == 0


def test_argument_checks_without_launch():
    lib = N.lib()
    assert lib.ls_inclusive_sum(7, None, None, 10, None, None, None, 0, None) == N.LS_ERR_UNSUPPORTED_DTYPE
    assert lib.ls_inclusive_sum(N.LS_I32, None, None, -1, None, None, None, 0, None) == N.LS_ERR_INVALID_ARG
    assert lib.ls_inclusive_sum(N.LS_I32, None, None, 5, None, None, None, 0, None) == N.LS_ERR_INVALID_ARG
    # partial overlap of x and y is rejected before anything touches a device
    buf = (ctypes.c_int32 * 64)()
    base = ctypes.addressof(buf)
    assert lib.ls_inclusive_sum(N.LS_I32, base, base + 4, 16, None, None, None, 0, None) == N.LS_ERR_INVALID_ARG
    assert "overlap" in N.last_detail()
    # misaligned element pointer
    assert lib.ls_inclusive_sum(N.LS_I32, base + 1, base + 129, 4, None, None, None, 0, None) == N.LS_ERR_INVALID_ARG
    assert lib.ls_carry_from_totals(N.LS_OP_ADD, N.LS_I32, None, 4, 0, None, None) == N.LS_ERR_INVALID_ARG
    assert lib.ls_inclusive_scan(7, N.LS_I32, None, None, 1, None, None, None, 0, None) == N.LS_ERR_UNSUPPORTED_DTYPE
    assert lib.ls_reduce(N.LS_OP_MAX, 9, None, 1, None, None, 0, None) == N.LS_ERR_UNSUPPORTED_DTYPE
    assert lib.ls_debug_config(0, -1, 0) == 0


def test_operator_surface():
    op = P.make_operator("add", "i32")
    assert op.identity == 0 and op.dtype == np.int32
    assert P.make_operator("max", "i64").identity == np.iinfo(np.int64).min
    with pytest.raises(P.UnsupportedOperatorError):
        P.make_operator("xor", "i32")
    with pytest.raises(P.UnsupportedOperatorError):
        P.parse_dtype("u32")
    assert issubclass(P.UnsupportedOperatorError, ValueError)
    assert P.make_operator("add", "i32").apply(2 ** 31 - 1, 1) == -2 ** 31


def test_problem_and_config_validation():
    with pytest.raises(P.ShapeError):
        P.ScanProblem(np.zeros((2, 2), dtype=np.int32), P.make_operator("add", "i32"))
    with pytest.raises(P.ShapeError):
        P.ScanProblem(np.zeros(4, dtype=np.int32), P.make_operator("add", "i32"),
                      out=np.zeros(3, dtype=np.int32))
    with pytest.raises(ValueError):
        P.ChainConfig(b=0)
    with pytest.raises(ValueError):
        P.ChainConfig(block_scan_mode="magic")
    with pytest.raises(ValueError):
        P.SpinPolicy(kind="nap")


def test_drop_in_rejects_before_device():
    x = np.arange(10, dtype=np.int32)

    class Xor:  # an operator the device does not implement
        name, dtype, identity = "xor", np.dtype(np.int32), 0

    with pytest.raises(P.UnsupportedOperatorError):
        P.chained_scan(P.ScanProblem(x, Xor()))
    with pytest.raises(P.ShapeError):  # dtype mismatch is refused, not guessed
        P.chained_scan(P.ScanProblem(x, P.make_operator("add", "i64")))
    # empty input: returns the output object untouched (chained.py:331-332)
    e = np.empty(0, dtype=np.int64)
    out = np.empty(0, dtype=np.int64)
    assert P.chained_scan(P.ScanProblem(e, P.make_operator("add", "i64"), out=out)) is out
    with pytest.raises(ValueError):
        P.run_algorithm("quantum", P.ScanProblem(x, P.make_operator("add", "i32")))


def test_shard_bounds():
    for n in (0, 1, 7, 1000, 2 ** 33):
        for world in (1, 2, 3, 8):
            bounds = [shard_bounds(n, world, r) for r in range(world)]
            assert bounds[0][0] == 0 and bounds[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(bounds, bounds[1:]))
            sizes = [hi - lo for lo, hi in bounds]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _build_c_demo(tmp_path):
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc unavailable")
    exe = tmp_path / "c_abi_demo"
    cmd = [gcc, "-O2", "-Wall", "-Werror", f"-I{N.INCLUDE}", "-I/usr/local/cuda/include",
           os.path.join(N.REPO_DIR, "examples", "c_abi_demo.c"), f"-L{N.LIB_DIR}", "-llscan",
           "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{N.LIB_DIR}", "-o", str(exe)]
    subprocess.run(cmd, check=True)
    return exe


def test_c_demo_compiles_against_the_header(tmp_path):
    # the ABI is consumable from plain C with the header alone
    assert _build_c_demo(tmp_path).exists()


@pytest.mark.gpu
def test_c_demo_runs(tmp_path):
    import subprocess
    exe = _build_c_demo(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c_abi_demo ok" in r.stdout


def test_every_module_imports():
    import importlib
    import pkgutil
    for m in pkgutil.iter_modules(P.__path__):
        if m.name == "__main__":
            continue
        importlib.import_module(f"paper_1604_04815_b200.{m.name}")


def test_torch_api_rejects_host_tensors():
    """No CPU fallback: host tensors are refused before anything is launched."""
    import torch
    from paper_1604_04815_b200 import scan as S
    x = torch.arange(10, dtype=torch.int32)
    with pytest.raises(ValueError, match="CUDA"):
        S.inclusive_scan(x)
    with pytest.raises(ValueError, match="CUDA"):
        S.exclusive_scan(x)
    with pytest.raises(P.ShapeError):
        S.inclusive_scan(torch.zeros(2, 2, dtype=torch.int32))
