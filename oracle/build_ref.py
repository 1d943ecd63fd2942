"""Recipe: byte-compile the reference package into oracle/_ref (test infrastructure only).

The reference (arxiv 2507.13681, /root/reference/pkg/src/loopserve) is pure
Python, so "building" it means compiling each module where it lies into a
sourceless `.pyc` under oracle/_ref/loopserve/ -- the Python analogue of a
`.so` built from the reference's own sources. No reference source text is
copied into this repository: oracle/_ref is git-ignored (it still travels to
the GPU box with the snapshot, like the built CUDA library), and the `.pyc`
files are the interpreter's compiled form of the unmodified sources.

Only `tests/` (the C1 run_turn drop-in parity test) imports it, as the
checker; the product package never does. Run by `__graft_entry__.build()`
when /root/reference is present; a no-op otherwise.

    python oracle/build_ref.py            # -> oracle/_ref/loopserve/*.pyc
"""

from __future__ import annotations

import glob
import os
import py_compile
import sys

REF_SRC = "/root/reference/pkg/src/loopserve"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref", "loopserve")


def build(src: str = REF_SRC, out: str = OUT) -> list[str]:
    if not os.path.isdir(src):
        return []
    os.makedirs(out, exist_ok=True)
    done = []
    for path in sorted(glob.glob(os.path.join(src, "*.py"))):
        name = os.path.splitext(os.path.basename(path))[0]
        cfile = os.path.join(out, name + ".pyc")
        # unchecked-hash pyc: valid without the source next to it (sourceless import)
        py_compile.compile(path, cfile=cfile, dfile=f"loopserve/{name}.py", doraise=True,
                           invalidation_mode=py_compile.PycInvalidationMode.UNCHECKED_HASH)
        done.append(cfile)
    with open(os.path.join(HERE, "_ref", "VERSION"), "w") as fh:
        import numpy as np

        fh.write(f"python {sys.version.split()[0]} numpy {np.__version__} from {src}\n")
    return done


def import_path() -> str | None:
    """sys.path entry that makes `import loopserve.*` load the compiled reference."""
    root = os.path.join(HERE, "_ref")
    return root if os.path.isfile(os.path.join(root, "loopserve", "session.pyc")) else None


if __name__ == "__main__":
    files = build()
    print(f"compiled {len(files)} reference modules into {OUT}" if files else "no /root/reference here: nothing built")
