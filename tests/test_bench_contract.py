"""bench.py keeps the driver's JSON contract (both arms)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def run(args, env=None, timeout=900):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=e, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.timeout(600)
def test_reference_arm_contract(ref_lib):
    """--impl reference: the reference library on the host cores, same workload and metric."""
    d = run(["--impl", "reference", "--steps", "2", "--warmup", "1", "--size", "32", "--sample-layers", "4"])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "entries/s"
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    # the reference's four methods with t_avg / t_min (bench.cpp:126-156, :223-224)
    assert set(d["config"]["methods"]) == {"spin-vec/crac", "colour-vec/crac", "atomic/csr", "seq/csr"}
    assert d["t_min_ms"] <= d["ms_per_step"]


@pytest.mark.gpu
@pytest.mark.timeout(900)
def test_gpu_arm_contract(gpu):
    d = run(["--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--size", "48"])
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["dtype"] == "f64" and d["higher_is_better"] is True
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1.2 and r["unit"] == "GB/s"
    assert d["gpu_launches"] == 3
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["e2e"]["values_equal_device_run"] is True
    assert d["clocks"]["sm_mhz"] is not None
    c = d["config"]
    assert c["soak_s"] == 0.0 and 0 < c["symbolic_phase_device_dofs_ms_rank0"] and 0 < c["symbolic_phase_ms_rank0"]


@pytest.mark.gpu
@pytest.mark.timeout(900)
def test_two_rank_partitioned_bench_matches_single_gpu(gpu):
    """torchrun, 2 ranks over gloo sharing the box's GPU: the row-partitioned path end to end;
    the gathered row blocks equal a single-GPU assembly of the global mesh bit for bit."""
    d = run(["--gpus", "2", "--steps", "2", "--warmup", "3", "--gather", "--check", "--size", "16",
             "--e2e-steps", "1"], env={"FEA_BENCH_BACKEND": "gloo", "MASTER_PORT": "29541"})
    assert d["n_gpus"] == 2 and d["gather"]["bitwise_equal_to_single_gpu"] is True
    assert d["scaling"] == "strong" and d["config"]["redundant_element_fraction"] > 0
    # every rank's host-path values equal its device-path values bit for bit
    assert d["e2e"]["values_equal_device_run"] is True
    # the fused path (each rank assembles into rank 0's buffer through a CUDA IPC mapping)
    assert d["gather"]["fused_equal_to_nccl_gather"] is True


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_config5_row_partition_tool_two_ranks(gpu):
    """tools/cfg5_ranks.py (BASELINE config 5 as a row-partitioned run) at reduced size, 2 ranks
    over gloo sharing the GPU: the fused assembly into rank 0's buffer equals a single-plan
    assembly of the whole mesh bit for bit."""
    e = dict(os.environ, FEA_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29543",
                        str(ROOT / "tools" / "cfg5_ranks.py"), "--size", "12", "--runs", "1", "--gather", "--check"],
                       capture_output=True, text=True, timeout=600, env=e, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["ranks"] == 2 and d["gathered_bitwise_equal_to_single_plan"] is True
    assert d["redundant_element_fraction"] > 0
