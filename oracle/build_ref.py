"""Recipe: build the UNMODIFIED reference package into ``oracle/_ref/`` (git-ignored).

The reference (``/root/reference/pkg/src/nfftkrr``) is pure Python, so "building" it
means byte-compiling its modules: this writes sourceless ``.pyc`` files into the zip
archive ``oracle/_ref/nfftkrr_ref.zip`` (``nfftkrr/*.pyc``, importable by zipimport
without the ``.py`` sources; a zip because the GPU-box snapshot skips loose ``.pyc``
files).  No source file is copied into the repository; the archive travels to the GPU
box with the snapshot (``oracle/_ref`` is listed in .gitignore but not in
.gpurunignore) and is what ``bench.py --impl reference`` times.  Run in the build
container:

    python oracle/build_ref.py          # (also run by __graft_entry__.build())
"""

from __future__ import annotations

import glob
import importlib.util
import marshal
import os
import sys
import zipfile

SRC = "/root/reference/pkg/src/nfftkrr"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref", "nfftkrr_ref.zip")


def _pyc(src):
    """Sourceless .pyc bytes (unchecked-hash header: no source needed to load it)."""
    with open(src, "rb") as fh:
        data = fh.read()
    code = compile(data, os.path.join("nfftkrr", os.path.basename(src)), "exec", dont_inherit=True)
    flags = (0b01).to_bytes(4, "little")            # hash-based, unchecked
    return importlib.util.MAGIC_NUMBER + flags + importlib.util.source_hash(data) + \
        marshal.dumps(code)


def build() -> str | None:
    if not os.path.isdir(SRC):
        return None          # GPU box: use the prebuilt oracle/_ref
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    tmp = OUT + ".tmp"
    with zipfile.ZipFile(tmp, "w", zipfile.ZIP_STORED) as z:
        for src in sorted(glob.glob(os.path.join(SRC, "*.py"))):
            z.writestr("nfftkrr/" + os.path.basename(src) + "c", _pyc(src))
        z.writestr("BUILD_INFO", f"compiled from {SRC} with Python {sys.version.split()[0]}\n")
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build())
