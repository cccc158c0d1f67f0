"""One-off stress run of the random-mesh parity test over many more seeds than the suite holds
(tests/test_gpu_parity.py::test_random_unstructured_meshes), plus the global-gather route on each.

    python tools/stress_random.py --seeds 400
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle as orc  # noqa: E402  (checker)
import paper_2012_00585_b200 as gpu  # noqa: E402
from tests.test_gpu_parity import test_random_unstructured_meshes as case  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seeds", type=int, default=200)
a = ap.parse_args()
orc.orc()
bad = 0
for env in ({}, {"FEA_GATHER_GLOBAL": "1"}, {"FEA_PLAN_NO_FUSED": "1"}):
    for k, v in env.items():
        os.environ[k] = v
    for seed in range(12, 12 + a.seeds):
        try:
            case(gpu, orc, seed)
        except Exception as e:  # noqa: BLE001
            bad += 1
            print("FAIL", env, seed, type(e).__name__, str(e)[:200], flush=True)
    for k in env:
        del os.environ[k]
    print("done", env, flush=True)
print("failures", bad)
sys.exit(1 if bad else 0)
