"""Build recipe for the oracle's C restatement -- TEST INFRASTRUCTURE ONLY.

Compiles ``oracle/ckernels.c`` into ``oracle/_build/liboracle.so`` with gcc.
Called from ``__graft_entry__.build()`` and lazily by ``oracle._native``.
"""

from __future__ import annotations

import os
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
SRC = HERE / "ckernels.c"
OUT = HERE / "_build" / "liboracle.so"


def build(force: bool = False) -> Path:
    if OUT.exists() and not force and OUT.stat().st_mtime >= SRC.stat().st_mtime:
        return OUT
    OUT.parent.mkdir(parents=True, exist_ok=True)
    tmp = OUT.with_suffix(f".{os.getpid()}.tmp")
    cmd = ["gcc", "-O3", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC",
           "-o", str(tmp), str(SRC), "-lm"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force=True))
