"""rnla_cli: the reference CLI's hot-path subcommands (tools/randnla_cli.cpp:127-445)
over the C ABI. RunReport schema (schemas/run_report.schema.json), exit codes
0 ok / 2 flagged / 1 error, Matrix Market / CSV parsing (src/io.cpp:47-230).
CPU tests cover argument handling and file parsing (which run before any
device work); GPU tests run every subcommand and check its metrics against
the oracle."""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1505_07570_b200", "_lib", "rnla_cli")

REQUIRED = {"command", "seed", "parameters", "metrics", "status"}


def run(*args, timeout=300):
    p = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=timeout)
    reports = [json.loads(line) for line in p.stdout.splitlines() if line.strip()]
    return p.returncode, reports, p.stderr


def check_schema(rep):
    assert REQUIRED <= set(rep) <= REQUIRED | {"elapsed_ms", "message"}
    assert isinstance(rep["seed"], int) and rep["seed"] >= 0
    assert all(isinstance(v, str) for v in rep["parameters"].values())
    assert all(isinstance(v, (int, float)) for v in rep["metrics"].values())
    assert rep["status"] in ("ok", "flagged", "error")
    assert list(rep["metrics"]) == sorted(rep["metrics"]) and list(rep["parameters"]) == sorted(rep["parameters"])


def save_mtx(path, m):
    m = np.atleast_2d(np.asarray(m, dtype=np.float64))
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix array real general\n% written by the test\n")
        f.write(f"{m.shape[0]} {m.shape[1]}\n")
        for v in m.T.reshape(-1):
            f.write(repr(float(v)) + "\n")


def save_csv(path, m):
    np.savetxt(path, np.atleast_2d(m), delimiter=",", fmt="%.17g")


def test_cli_argument_errors():
    assert os.path.exists(CLI)
    assert run()[0] == 106
    assert run("sketch", "--s", "3", "--seed", "1")[0] == 106              # --input missing
    assert run("sketch", "--input", "/nonexistent.mtx", "--s", "3", "--seed", "1")[0] == 105
    assert run("sketch", "--bogus", "1")[0] == 109
    assert run("verify", "--s", "3")[0] == 109                             # not part of this build


def test_cli_parse_errors_are_reports(tmp_path):
    bad = tmp_path / "bad.mtx"
    bad.write_text("%%MatrixMarket matrix array real general\n2 2\n1\n2\nx\n4\n")
    code, reps, _ = run("sketch", "--input", bad, "--s", "2", "--seed", "3")
    assert code == 1 and len(reps) == 1
    check_schema(reps[0])
    assert reps[0]["status"] == "error" and reps[0]["message"].endswith(":5: malformed value")
    assert reps[0]["metrics"] == {}
    short = tmp_path / "short.csv"
    short.write_text("1,2\n3\n")
    code, reps, _ = run("nystrom", "--data", short, "--sigma", "1", "--seed", "3")
    assert code == 1 and reps[0]["message"].endswith(":2: row has 1 cells, expected 2")
    cnt = tmp_path / "cnt.mtx"
    cnt.write_text("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n2 2 2.0\n")
    code, reps, _ = run("sketch", "--input", cnt, "--s", "2", "--seed", "3")
    assert "entry count mismatch: header says 3, file has 2" in reps[0]["message"]


def test_cli_lsr_requires_seed_for_randomized(tmp_path):
    save_mtx(tmp_path / "a.mtx", orc.gaussian_matrix(20, 3, 1))
    save_mtx(tmp_path / "b.mtx", orc.gaussian_matrix(20, 1, 2))
    code, reps, _ = run("lsr", "--method", "sketched", "--input", tmp_path / "a.mtx", "--rhs", tmp_path / "b.mtx")
    assert code == 1 and reps[0]["message"] == "--seed is required for --method sketched"
    check_schema(reps[0])


@pytest.mark.gpu
def test_cli_sketch_and_lsr(tmp_path):
    a = orc.gaussian_matrix(300, 8, 5)
    b = a @ orc.gaussian_matrix(8, 1, 6)[:, 0] + 0.1 * orc.gaussian_matrix(300, 1, 7)[:, 0]
    save_mtx(tmp_path / "a.mtx", a)
    save_csv(tmp_path / "b.csv", b[:, None])
    code, reps, _ = run("sketch", "--input", tmp_path / "a.mtx", "--method", "gaussian", "--s", "5", "--seed", "9",
                        "--output", tmp_path / "c.mtx")
    assert code == 0
    rep = reps[0]
    check_schema(rep)
    c = orc.gaussian_sketch(a, 5, 9)
    assert abs(rep["metrics"]["sketch_fro"] - np.linalg.norm(c)) <= 1e-10 * np.linalg.norm(c)
    assert rep["metrics"]["sketch_cols"] == 5 and rep["parameters"] == {"input": str(tmp_path / "a.mtx"),
                                                                        "method": "gaussian", "s": "5"}
    exact = np.linalg.lstsq(a, b, rcond=None)[0]
    obj = float(np.sum((a @ exact - b) ** 2))
    for method, extra in [("exact", []), ("cg", ["--tol", "1e-12"]), ("preconditioned", ["--seed", "3", "--eps", "1e-10"]),
                          ("sketched", ["--seed", "3", "--sketch-size", "100"])]:
        code, reps, _ = run("lsr", "--method", method, "--input", tmp_path / "a.mtx", "--rhs", tmp_path / "b.csv",
                            *extra, "--output", tmp_path / "x.csv")
        assert code == 0, reps
        check_schema(reps[0])
        if method != "sketched":
            assert abs(reps[0]["metrics"]["objective"] - obj) <= 1e-9 * obj
            x = np.loadtxt(tmp_path / "x.csv", delimiter=",")
            assert np.allclose(x, exact, rtol=1e-8, atol=1e-10)
        else:
            assert obj - 1e-9 <= reps[0]["metrics"]["objective"] <= 1.5 * obj
        # kappa is reported only when the solver estimates it (preconditioned),
        # as the reference CLI's `if (sol.kappa_estimate)` (tools/randnla_cli.cpp:303-304)
        assert ("kappa" in reps[0]["metrics"]) == (method == "preconditioned"), (method, reps[0]["metrics"])


@pytest.mark.gpu
def test_cli_ksvd_spsd_nystrom(tmp_path):
    a = orc.gaussian_matrix(120, 4, 6) @ orc.gaussian_matrix(4, 100, 60)
    save_mtx(tmp_path / "a.mtx", a)
    for method in ("prototype", "faster"):
        code, reps, _ = run("ksvd", "--method", method, "--input", tmp_path / "a.mtx", "--k", "4", "--seed", "9")
        assert code == 0, reps
        check_schema(reps[0])
        m = reps[0]["metrics"]
        assert m["passes"] == 2 and m["error_fro"] <= 1e-6 * np.linalg.norm(a)
        assert abs(m["top_sv"] - np.linalg.svd(a, compute_uv=False)[0]) <= 1e-8 * m["top_sv"]
    code, reps, _ = run("ksvd", "--method", "lanczos", "--input", tmp_path / "a.mtx", "--k", "4", "--seed", "9")
    assert code == 1 and reps[0]["status"] == "error"
    x = orc.gaussian_matrix(150, 3, 2)
    save_csv(tmp_path / "x.csv", x)
    code, reps, _ = run("nystrom", "--data", tmp_path / "x.csv", "--sigma", "2", "--l", "40", "--seed", "4")
    assert code == 0
    L, _, _ = orc.nystrom(x, 2.0, 40, 4, 0)
    k = orc.rbf_kernel(x, x, 2.0)
    err = np.linalg.norm(k - L @ L.T) / np.linalg.norm(k)
    assert abs(reps[0]["metrics"]["error_rel"] - err) <= 1e-6 * max(err, 1e-12)
    assert reps[0]["metrics"]["rank"] == L.shape[1]
    code, reps, _ = run("spsd", "--data", tmp_path / "x.csv", "--sigma", "2", "--s", "10", "--p", "40", "--seed", "6")
    assert code in (0, 2)
    check_schema(reps[0])
    q, z, sel, sec, flagged = orc.spsd_faster(x, 2.0, 10, 40, 6)
    err = np.linalg.norm(k - q @ z @ q.T) / np.linalg.norm(k)
    assert abs(reps[0]["metrics"]["error_rel"] - err) <= 1e-8
    assert reps[0]["metrics"]["kernel_entries"] == 150 * 10 + len(sec) ** 2
    code, reps, _ = run("spsd", "--method", "prototype", "--data", tmp_path / "x.csv", "--sigma", "2", "--s", "10",
                        "--seed", "6")
    assert code == 0 and 0.0 <= reps[0]["metrics"]["error_rel"] < 1.0


@pytest.mark.gpu
def test_cli_cur_kernel(tmp_path):
    xtest = orc.gaussian_matrix(45, 3, 15)
    xtrain = orc.gaussian_matrix(60, 3, 16)
    save_csv(tmp_path / "te.csv", xtest)
    save_csv(tmp_path / "tr.csv", xtrain)
    code, reps, _ = run("cur", "--train", tmp_path / "tr.csv", "--test", tmp_path / "te.csv", "--sigma", "1.3",
                        "--c", "7", "--r", "6", "--seed", "17", "--output", tmp_path / "cur.mtx")
    assert code in (0, 2), reps
    check_schema(reps[0])
    ks = orc.rbf_kernel(xtest, xtrain, 1.3)
    C, U, R, ci, ri, pc, pr, flagged = orc.cur_faster(ks, 7, 6, 17)
    m = reps[0]["metrics"]
    assert m["core_rows"] == 7 and m["core_cols"] == 6
    assert m["entries_visited"] == 45 * 7 + 6 * 60 + len(pc) * len(pr)
    code, reps, _ = run("cur", "--input", tmp_path / "tr.csv", "--c", "2", "--r", "2", "--seed", "1")
    assert code == 1 and "not part of the B200 hot path" in reps[0]["message"]
