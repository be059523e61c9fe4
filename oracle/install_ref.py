"""Install the UNMODIFIED reference package (`vrlab`, pure Python + NumPy) into oracle/_ref/ so that bench.py's
reference arm can time the reference's own `run_on_indices` on the GPU box's host cores (SURVEY.md 8d "CPU
baseline").  TEST / MEASUREMENT INFRASTRUCTURE ONLY: nothing under paper_1805_08893_b200/ imports it.

    python oracle/install_ref.py        # needs /root/reference (this container); a no-op elsewhere

The install is the contract's offline pip install (no index, no build isolation, no dependencies) from a scratch
copy of the source tree (/root/reference is read-only).  oracle/_ref/ is git-ignored -- no reference source enters
the history -- but not gpurun-ignored, so it travels to the GPU box like the built .so files."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
TARGET = os.path.join(HERE, "_ref")
SOURCE = "/root/reference/pkg"


def installed() -> bool:
    return os.path.exists(os.path.join(TARGET, "vrlab", "strategies.py"))


def install(force: bool = False) -> bool:
    """True if oracle/_ref holds the reference afterwards."""
    if installed() and not force:
        return True
    if not os.path.isdir(SOURCE):
        return installed()
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(SOURCE, src)
        cmd = [sys.executable, "-m", "pip", "install", "--quiet", "--no-index", "--no-build-isolation", "--no-deps",
               "--find-links", "/opt/wheelhouse", "--upgrade", "--target", TARGET, src]
        subprocess.check_call(cmd)
    return installed()


if __name__ == "__main__":
    print("oracle/_ref:", "installed" if install(force="--force" in sys.argv) else "unavailable (no /root/reference)")
