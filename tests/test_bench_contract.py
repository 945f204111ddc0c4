"""bench.py contract checks that need no GPU: `--impl reference` (the CPU oracle arm) prints
exactly ONE JSON line on stdout with the contract's keys, even when libraries write to fd 1."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_contract_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "C1", "--steps", "1",
                        "--warmup", "0"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["higher_is_better"] is True and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("C1")


def test_stdout_is_private_to_the_json_line():
    # a C-level write to fd 1 after bench's redirection lands on stderr, not stdout
    code = ("import bench, os; bench._private_stdout(); os.write(1, b'BANNER\\n'); print('{\"ok\": 1}')")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == '{"ok": 1}'
    assert "BANNER" in r.stderr


def test_exact_len_sum_matches_golden_counts():
    """bench.exact_len_sum (closed form per sweep) equals the enumerated sum L of
    tests/golden/paper_counts.txt for C1-C5 (exact flops = 4 sum L nev)."""
    sys.path.insert(0, ROOT)
    import bench
    for line in open(os.path.join(ROOT, "tests", "golden", "paper_counts.txt")):
        if line.startswith("#") or not line.strip():
            continue
        name, n, b, nev, R, sumL = line.split()
        assert bench.exact_len_sum(int(n), int(b)) == int(sumL), name
    assert bench.exact_len_sum(2, 8) == 0 and bench.exact_len_sum(100, 1) == 0
