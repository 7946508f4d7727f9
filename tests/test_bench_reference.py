"""`bench.py --impl reference` (the CPU oracle arm) runs on the CPU and
prints one JSON line with the contract's keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref_line(*extra):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config",
                          "uniform2k_k8", "--steps", "2", "--warmup", "1", *extra],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    return json.loads(lines[0])


def test_reference_arm_whole_matrix_config():
    """When the oracle finishes the whole matrix within the budget, the
    reference line's config is the GPU arm's config of the same workload."""
    sys.path.insert(0, ROOT)
    import bench
    import oracle
    d = _ref_line()
    assert d["cpu_baseline"]["sample"].startswith("whole matrix")
    A, B, desc = bench.build_workload("uniform2k_k8", 1)
    C = oracle.spgemm_gustavson(A, B)
    nprod = int(oracle.row_nprod(A, B).sum())
    want = bench.workload_config("uniform2k_k8", desc, "upper", A, nprod, int(C.rpt[-1]))
    assert d["config"] == json.loads(json.dumps(want))


def test_reference_arm_sampled():
    d = _ref_line("--ref-budget-s", "0.0003")
    assert "evenly strided" in d["cpu_baseline"]["sample"] and d["config"]["rows_sampled"] < 2000


def test_reference_arm_json():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config",
                          "uniform2k_k8", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e", "impl", "dtype"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GFLOP/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"] == "uniform2k_k8"


def test_reference_arm_nonzero_rank_is_silent():
    env = dict(os.environ, RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config",
                          "uniform2k_k8", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""
