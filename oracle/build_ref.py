"""Recipe: byte-compile the reference package into oracle/_ref (test infrastructure only).

The reference (arxiv 2507.13681, /root/reference/pkg/src/loopserve) is pure
Python, so "building" it means compiling each module where it lies into
sourceless bytecode (a `.pyc` image, stored as `<module>.refbc` so snapshot
tools that drop `*.pyc` still ship it) under oracle/_ref/loopserve/ -- the
Python analogue of a `.so` built from the reference's own sources. No reference source text is
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
SUFFIX = ".refbc"
OUT = os.path.join(HERE, "_ref", "loopserve")


def build(src: str = REF_SRC, out: str = OUT) -> list[str]:
    if not os.path.isdir(src):
        return []
    os.makedirs(out, exist_ok=True)
    done = []
    for path in sorted(glob.glob(os.path.join(src, "*.py"))):
        name = os.path.splitext(os.path.basename(path))[0]
        cfile = os.path.join(out, name + SUFFIX)
        # unchecked-hash pyc: valid without the source next to it (sourceless import)
        py_compile.compile(path, cfile=cfile, dfile=f"loopserve/{name}.py", doraise=True,
                           invalidation_mode=py_compile.PycInvalidationMode.UNCHECKED_HASH)
        done.append(cfile)
    with open(os.path.join(HERE, "_ref", "VERSION"), "w") as fh:
        import numpy as np

        fh.write(f"python {sys.version.split()[0]} numpy {np.__version__} from {src}\n")
    return done


class _RefFinder:
    """meta-path finder: `loopserve` (namespace) and `loopserve.<m>` from the
    compiled bytecode in oracle/_ref/loopserve."""

    def __init__(self, root: str):
        self.root = root

    def find_spec(self, fullname, path=None, target=None):
        import importlib.machinery as M
        import importlib.util as U

        if fullname == "loopserve":
            spec = M.ModuleSpec("loopserve", None, is_package=True)
            spec.submodule_search_locations = [os.path.join(self.root, "loopserve")]
            return spec
        if fullname.startswith("loopserve."):
            f = os.path.join(self.root, "loopserve", fullname.split(".", 1)[1] + SUFFIX)
            if os.path.isfile(f):
                return U.spec_from_loader(fullname, M.SourcelessFileLoader(fullname, f))
        return None


def install_import(root: str | None = None) -> bool:
    """Make `import loopserve.*` load the compiled reference; False if absent."""
    root = root or os.path.join(HERE, "_ref")
    if not os.path.isfile(os.path.join(root, "loopserve", "session" + SUFFIX)):
        return False
    if not any(isinstance(f, _RefFinder) for f in sys.meta_path):
        sys.meta_path.insert(0, _RefFinder(root))
    return True


if __name__ == "__main__":
    files = build()
    print(f"compiled {len(files)} reference modules into {OUT}" if files else "no /root/reference here: nothing built")
