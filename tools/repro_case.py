"""Run one golden case under every workflow (for compute-sanitizer repros):
python tools/repro_case.py NAME"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from golden_io import Case  # noqa: E402
from paper_2604_19004_b200 import EngineConfig, WorkflowOverride, spgemm  # noqa: E402

c = Case(sys.argv[1])
for o in WorkflowOverride:
    C, rep = spgemm(c.A, c.B, EngineConfig(workflow=o, tiers=c.tiers() or EngineConfig().tiers))
    c.check_product(C)
    print(o, "ok", flush=True)
