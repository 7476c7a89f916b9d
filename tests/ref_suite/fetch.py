"""Stage the reference's own hot-path test files for the import-shim run (test infrastructure).

The reference package (`/root/reference/pkg`) is pure Python and does not travel to the
GPU box.  This script copies, UNMODIFIED, the reference test modules that exercise the
hot path (transforms, coding, history/dictionary, training, acceptance criteria) plus the
two helper modules those tests import that are not on the path (`synthetic.py`, the data
generator, and `baselines.py`, the dense/FISTA comparators of acceptance 6) into
`tests/ref_suite/_ref/`.  That directory is git-ignored (it never enters history, like
`oracle/_ref/`) but not gpurun-ignored, so it ships to the B200 box with the snapshot;
`tests/ref_suite/conftest.py` then runs the tests against `paper_1706_06972_b200` through
the `ocsc` shim package in `tests/ref_suite/shim/`.

Run by `__graft_entry__.build()` whenever `/root/reference` exists.
"""

from __future__ import annotations

import os
import shutil
import sys

REF = "/root/reference/pkg"
HERE = os.path.dirname(os.path.abspath(__file__))
DEST = os.path.join(HERE, "_ref")

TESTS = ["test_transforms.py", "test_coding.py", "test_dictionary.py", "test_training.py",
         "test_acceptance.py"]
HELPERS = ["synthetic.py", "baselines.py"]   # loaded by the shim's ocsc.synthetic / ocsc.baselines


def fetch(ref: str = REF, dest: str = DEST) -> bool:
    if not os.path.isdir(os.path.join(ref, "tests")):
        return False
    os.makedirs(dest, exist_ok=True)
    for name in TESTS:
        shutil.copyfile(os.path.join(ref, "tests", name), os.path.join(dest, name))
    for name in HELPERS:
        shutil.copyfile(os.path.join(ref, "src", "ocsc", name), os.path.join(dest, "ref_" + name))
    with open(os.path.join(dest, "__init__.py"), "w") as f:
        f.write("# reference tests staged by tests/ref_suite/fetch.py (git-ignored)\n")
    return True


if __name__ == "__main__":
    ok = fetch()
    print("staged reference tests into", DEST if ok else "(reference not present)")
    sys.exit(0)
