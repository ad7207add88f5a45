"""Build the sm_100a extension in-tree (lib/libkvtier_b200.so) with nvcc via csrc/Makefile."""

from __future__ import annotations

import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB = PKG / "lib" / "libkvtier_b200.so"


def build(jobs: int | None = None, force: bool = False) -> Path:
    jobs = jobs or max(1, min(8, os.cpu_count() or 1))
    if force:
        subprocess.run(["make", "-s", "-C", str(PKG / "csrc"), "clean"], check=True)
    subprocess.run(["make", "-s", "-C", str(PKG / "csrc"), f"-j{jobs}"], check=True)
    if not LIB.exists():
        raise RuntimeError(f"build did not produce {LIB}")
    return LIB


if __name__ == "__main__":
    print(build())
