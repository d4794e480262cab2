"""Recipe: build the UNMODIFIED reference package into ``oracle/_ref/`` (git-ignored).

The reference (``/root/reference/pkg/src/nfftkrr``) is pure Python, so "building" it
means byte-compiling its modules: this writes sourceless ``.pyc`` files (legacy layout,
importable without the ``.py`` sources) to ``oracle/_ref/nfftkrr/``.  No source file is
copied into the repository; the compiled package travels to the GPU box with the
snapshot (``oracle/_ref`` is listed in .gitignore but not in .gpurunignore) and is what
``bench.py --impl reference`` times.  Run in the build container:

    python oracle/build_ref.py          # (also run by __graft_entry__.build())
"""

from __future__ import annotations

import glob
import os
import py_compile
import sys

SRC = "/root/reference/pkg/src/nfftkrr"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref", "nfftkrr")


def build() -> str | None:
    if not os.path.isdir(SRC):
        return None          # GPU box: use the prebuilt oracle/_ref
    os.makedirs(OUT, exist_ok=True)
    for src in sorted(glob.glob(os.path.join(SRC, "*.py"))):
        name = os.path.basename(src)[:-3]
        py_compile.compile(src, cfile=os.path.join(OUT, name + ".pyc"), doraise=True,
                           invalidation_mode=py_compile.PycInvalidationMode.UNCHECKED_HASH)
    with open(os.path.join(OUT, "BUILD_INFO"), "w") as fh:
        fh.write(f"compiled from {SRC} with Python {sys.version.split()[0]}\n")
    return OUT


if __name__ == "__main__":
    print(build())
