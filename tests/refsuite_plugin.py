"""pytest plugin (-p refsuite_plugin): before the reference's test modules
are imported, route ``sketchgemm.spgemm`` to the B200 path through
``paper_2604_19004_b200.refbind`` (the reference-side binding of
INTEGRATION.md §2).  Used by tests/test_gpu_reference_suite.py."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
for p in (os.path.join(REF, "reference_tests"), REF, ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)

import sketchgemm  # noqa: E402  (the unmodified reference package)

from paper_2604_19004_b200 import refbind  # noqa: E402

refbind.install(sketchgemm)
assert sketchgemm.spgemm.__module__ == "paper_2604_19004_b200.refbind"
