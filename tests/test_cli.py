"""The CLI's exit-code contract and report schemas (tools/mih.cpp:28-31, tests/cli_smoke.sh).
CPU: usage and data errors; GPU: the full gen/build/query/benchmark round."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, cwd):
    return subprocess.run([sys.executable, "-m", "paper_1307_2982_b200.cli", *args], cwd=cwd,
                          capture_output=True, text=True, env={**os.environ, "PYTHONPATH": ROOT})


def test_cli_usage_and_data_errors(tmp_path):
    assert run([], tmp_path).returncode == 1                          # no subcommand
    assert run(["query", "--index", "idx.bin"], tmp_path).returncode == 1  # missing option
    assert run(["build", "--dataset", "/nonexistent/x.bin", "--out", "y.bin"], tmp_path).returncode == 2
    (tmp_path / "bad.bin").write_bytes(b"corrupt")
    r = run(["build", "--dataset", "bad.bin", "--out", "y.bin"], tmp_path)
    assert r.returncode == 2 and "format error" in r.stderr


def test_cli_gen_is_deterministic(tmp_path):
    assert run(["gen", "--mode", "uniform", "--n", "500", "--bits", "70", "--seed", "11", "--out", "a.bin"], tmp_path).returncode == 0
    assert run(["gen", "--mode", "uniform", "--n", "500", "--bits", "70", "--seed", "11", "--out", "b.bin"], tmp_path).returncode == 0
    assert (tmp_path / "a.bin").read_bytes() == (tmp_path / "b.bin").read_bytes()
    assert run(["gen", "--mode", "correlated", "--n", "300", "--bits", "32", "--block", "4", "--seed", "13",
                "--out", "c.bin"], tmp_path).returncode == 0


def test_cli_correlated_matches_reference(tmp_path):
    """gen --mode correlated == the reference's gen_duplicated_bits (io.hpp:281-297)."""
    import oracle

    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    import numpy as np

    sys.path.insert(0, ROOT)
    from paper_1307_2982_b200.cli import gen_duplicated_bits

    got = gen_duplicated_bits(400, 96, 3, 77).raw_words()
    import ctypes as C

    R = oracle.ref()
    assert hasattr(R.lib, "ref_gen_duplicated")
    out = np.zeros(400 * 2, np.uint64)
    R.lib.ref_gen_duplicated.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, oracle._u64p]
    assert R.lib.ref_gen_duplicated(400, 96, 3, 77, out.ctypes.data_as(oracle._u64p)) == 0
    assert np.array_equal(got, out.reshape(400, 2))


@pytest.mark.gpu
def test_cli_end_to_end(cuda_ok, tmp_path):
    for args in (["gen", "--mode", "uniform", "--n", "20000", "--bits", "64", "--seed", "11", "--out", "data.bin"],
                 ["gen", "--mode", "uniform", "--n", "200", "--bits", "64", "--seed", "12", "--out", "q.bin"],
                 ["gen", "--mode", "uniform", "--n", "50", "--bits", "32", "--seed", "13", "--out", "q32.bin"],
                 ["build", "--dataset", "data.bin", "--out", "idx.bin"],
                 ["build", "--dataset", "data.bin", "--tables", "4", "--stats", "--out", "idx4.bin"],
                 ["query", "--index", "idx.bin", "--queries", "q.bin", "--k", "5", "--out", "knn.csv"],
                 ["query", "--index", "idx.bin", "--queries", "q.bin", "--radius", "8", "--format", "json",
                  "--out", "range.json"],
                 ["benchmark", "--dataset", "data.bin", "--queries", "q.bin", "--k", "3", "--radius", "6",
                  "--warmup", "5", "--out", "bench.csv"],
                 ["benchmark", "--dataset", "data.bin", "--queries", "q.bin", "--k", "3", "--format", "json",
                  "--out", "bench.json"]):
        r = run(args, tmp_path)
        assert r.returncode == 0, (args, r.stderr)
    assert (tmp_path / "knn.csv").read_text().splitlines()[0] == "query,rank,id,dist"
    assert len(json.load(open(tmp_path / "range.json"))) == 200
    csv = (tmp_path / "bench.csv").read_text()
    assert "\nmih,k,3," in csv and "\nscan,r,6," in csv
    rows = json.load(open(tmp_path / "bench.json"))["rows"]
    assert any(r["method"] == "mih" and r["speedup_vs_scan"] > 0 for r in rows)
    need = {"mean_us", "median_us", "p95_us", "mean_lookups", "mean_unique_candidates"}
    assert all(need <= set(r) for r in rows)
    assert run(["query", "--index", "idx.bin", "--queries", "q.bin", "--k", "2", "--radius", "3"], tmp_path).returncode == 1
    assert run(["query", "--index", "idx.bin", "--queries", "q32.bin", "--k", "2"], tmp_path).returncode == 2


@pytest.mark.gpu
def test_cli_optimize_then_build(cuda_ok, tmp_path):
    """optimize (tools/mih.cpp:502-512) writes a partition JSON that build --partition accepts; on
    block-correlated codes it separates every duplicated block (optimize_test.cpp:87-102)."""
    assert run(["gen", "--mode", "correlated", "--n", "3000", "--bits", "16", "--block", "2", "--seed", "21",
                "--out", "dup.bin"], tmp_path).returncode == 0
    r = run(["optimize", "--dataset", "dup.bin", "--tables", "4", "--seed", "77", "--out", "part.json"], tmp_path)
    assert r.returncode == 0, r.stderr
    j = json.load(open(tmp_path / "part.json"))
    assert j["bits"] == 16 and len(j["substrings"]) == 4
    assert all(len({x // 2 for x in s}) == len(s) == 4 for s in j["substrings"])
    r = run(["build", "--dataset", "dup.bin", "--partition", "part.json", "--out", "idx.bin"], tmp_path)
    assert r.returncode == 0, r.stderr
    assert run(["optimize", "--dataset", "missing.bin", "--out", "p.json"], tmp_path).returncode == 2
