"""Stage the reference package (its source and its own tests) into
``oracle/_ref/pkg`` — TEST INFRASTRUCTURE, never imported by the product.

``/root/reference`` exists only in the build container; the GPU box gets the
staged copy with the repo snapshot (``oracle/_ref/`` is git-ignored, so no
reference source enters history, but it is not gpurun-ignored, so it
travels).  ``tests/test_reference_suite_gpu.py`` runs the reference's own
chained-scan tests from it with ``chainscan.chained_scan`` swapped for the
GPU drop-in.  Plain file copies; nothing is built or installed.

    python oracle/stage_reference.py [--src /root/reference/pkg]
"""

from __future__ import annotations

import argparse
import os
import shutil

HERE = os.path.dirname(os.path.abspath(__file__))
DEST = os.path.join(HERE, "_ref", "pkg")


def stage(src: str = "/root/reference/pkg") -> bool:
    if not os.path.isdir(os.path.join(src, "src", "chainscan")):
        return False
    if os.path.isdir(DEST):
        shutil.rmtree(DEST)
    ignore = shutil.ignore_patterns("__pycache__", "*.pyc", ".pytest_cache")
    shutil.copytree(os.path.join(src, "src", "chainscan"), os.path.join(DEST, "src", "chainscan"), ignore=ignore)
    shutil.copytree(os.path.join(src, "tests"), os.path.join(DEST, "tests"), ignore=ignore)
    for f in ("pyproject.toml", "README.md"):
        if os.path.exists(os.path.join(src, f)):
            shutil.copy2(os.path.join(src, f), os.path.join(DEST, f))
    return True


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--src", default="/root/reference/pkg")
    ok = stage(ap.parse_args().src)
    print("staged" if ok else "reference not found; nothing staged")
