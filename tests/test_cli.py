"""The `sfdg` CLI (tools/sfdg_main.cpp): the reference's four commands (tools/sfd_main.cpp).

CPU tests: `generate` byte for byte against the reference generator (oracle/_ref/refio --gen,
and the committed SHA-256 fixture where the reference is absent), manifests, and the argument /
input errors that fail before any device work (exit 1, the reference's messages). GPU tests:
`eval` and `bench` metric values against the oracle's exact_tail / proj_err / cov_err with the
reference's seed plumbing (sfd_main.cpp:123-155, 157-228; bench.cpp:185-237).
"""
import hashlib
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tools", "sfdg")
REFIO = os.path.join(ROOT, "oracle", "_ref", "refio")
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "cli_generate_golden.json")))


@pytest.fixture(scope="module")
def sfdg():
    if not os.path.exists(EXE):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tools"), "sfdg"], check=True, capture_output=True)
    return EXE


def run(*args):
    return subprocess.run([EXE, *map(str, args)], capture_output=True, text=True)


# ---------------------------------------------------------------- generate (CPU)
@pytest.mark.parametrize("spec", GOLD, ids=lambda s: f"n{s['n']}d{s['d']}z{s['z']}s{s['seed']}")
def test_generate_matches_reference_bytes(sfdg, tmp_path, spec):
    """SyntheticStream (bench.cpp:27-66) through MatrixMarketWriter (io.cpp:200-230): the same
    file as the reference for the same (n, d, z, seed) -- pinned by the fixture's SHA-256, and
    against the compiled reference itself when present."""
    out = tmp_path / "g.mtx"
    r = run("generate", "--n", spec["n"], "--d", spec["d"], "--z", spec["z"], "--seed", spec["seed"],
            "--output", out)
    assert r.returncode == 0, r.stderr
    data = out.read_bytes()
    assert len(data) == spec["bytes"]
    assert hashlib.sha256(data).hexdigest() == spec["sha256"]
    if os.path.exists(REFIO):
        ref = tmp_path / "r.mtx"
        subprocess.run([REFIO, "--gen", str(spec["n"]), str(spec["d"]), str(spec["z"]), str(spec["seed"]), str(ref)],
                       check=True)
        assert ref.read_bytes() == data


def test_generate_rows_and_manifest(sfdg, tmp_path):
    """Every row has exactly z distinct sorted columns with +-1 values, ~90% of the entries in
    the ceil(1.5 z)-column head; the manifest carries the reference's keys, sorted."""
    import paper_1602_00412_b200 as P
    out = tmp_path / "g.mtx"
    n, d, z = 3000, 400, 20
    assert run("generate", "--n", n, "--d", d, "--z", z, "--seed", 5, "--output", out).returncode == 0
    rp, cs, vs, dd = P.read_row_stream(str(out))
    assert dd == d and len(rp) == n + 1 and np.all(np.diff(rp) == z)
    assert set(np.unique(vs)) == {-1.0, 1.0}
    for i in range(0, n, 97):
        row = cs[rp[i]:rp[i + 1]]
        assert np.all(np.diff(row.astype(np.int64)) > 0)
    head_share = float((cs < 30).mean())
    assert 0.88 < head_share < 0.92
    text = open(str(out) + ".manifest.json").read()
    man = json.loads(text)
    assert list(man) == sorted(man)
    assert man == {"command": "generate", "version": man["version"], "output": str(out), "n": n, "d": d, "z": z,
                   "p_head": 0.9, "seed": 5}
    assert '"p_head": 0.9,' in text and text.startswith("{\n  \"command\"")


def test_generate_defaults_shape(sfdg, tmp_path):
    """Defaults n = 10000, d = 1000, z = 100, seed 0 (sfd_main.cpp:245-252): header line."""
    out = tmp_path / "g.mtx"
    assert run("generate", "--output", out).returncode == 0
    with open(out) as f:
        assert f.readline() == "%%MatrixMarket matrix coordinate real general\n"
        assert f.readline() == "10000 1000 1000000\n"


# ---------------------------------------------------------------- errors (CPU)
def test_cli_usage_errors(sfdg, tmp_path):
    """Parse errors exit 1 (CLI11 ParseError -> 1, sfd_main.cpp:285-288); --help exits 0."""
    assert run("--help").returncode == 0
    assert run("generate", "--help").returncode == 0
    for args in ((), ("frobnicate",), ("generate",), ("generate", "--output"), ("generate", "--bogus", "1"),
                 ("generate", "--n", "x", "--output", tmp_path / "a"), ("sketch", "--input", "a", "--output", "b"),
                 ("sketch", "--input", "a", "--output", "b", "--ell", "5", "--algo", "svd"),
                 ("bench", "--sweep", "q", "--out-csv", tmp_path / "b.csv"), ("eval", "--matrix", "a")):
        r = run(*args)
        assert r.returncode == 1, (args, r.stderr)


def test_cli_invalid_inputs(sfdg, tmp_path):
    """std::invalid_argument paths exit 1 with the reference's message (sfd_main.cpp:293-296),
    all raised before any device work."""
    r = run("generate", "--n", 3, "--d", 2, "--z", 3, "--output", tmp_path / "g.mtx")
    assert r.returncode == 1 and "SyntheticSpec: requires 1 <= z <= d" in r.stderr
    mtx = tmp_path / "a.mtx"
    assert run("generate", "--n", 20, "--d", 8, "--z", 3, "--output", mtx).returncode == 0
    bad = tmp_path / "bad.csv"
    bad.write_text("1,2,3\n")
    r = run("eval", "--matrix", mtx, "--sketch", bad, "--output", tmp_path / "m.csv")
    assert r.returncode == 1 and "eval: matrix and sketch dimensions are incompatible" in r.stderr
    bad.write_text("1,2,3,4,5,6,7,8\n1,2\n")
    r = run("eval", "--matrix", mtx, "--sketch", bad, "--output", tmp_path / "m.csv")
    assert r.returncode == 1 and "ragged sketch file" in r.stderr
    bad.write_text("\n\n")
    r = run("eval", "--matrix", mtx, "--sketch", bad, "--output", tmp_path / "m.csv")
    assert r.returncode == 1 and "empty sketch file" in r.stderr
    r = run("eval", "--matrix", mtx, "--sketch", tmp_path / "none.csv", "--output", tmp_path / "m.csv")
    assert r.returncode == 1 and "cannot open sketch file" in r.stderr
    r = run("eval", "--matrix", tmp_path / "none.mtx", "--sketch", bad, "--output", tmp_path / "m.csv")
    assert r.returncode == 1
    plain = tmp_path / "p.txt"
    plain.write_text("0:1 3:2\n")
    r = run("sketch", "--input", plain, "--output", tmp_path / "s.csv", "--ell", 2)
    assert r.returncode == 1 and "explicit column count" in r.stderr


# ---------------------------------------------------------------- eval / bench (GPU)
def _metrics(path):
    lines = open(path).read().splitlines()
    assert lines[0] == "algo,n,d,ell,z,k,proj_err,cov_err,wall_seconds,seed"
    rows = []
    for ln in lines[1:]:
        f = ln.split(",")
        rows.append({"algo": f[0], "n": int(f[1]), "d": int(f[2]), "ell": int(f[3]), "z": int(f[4]), "k": int(f[5]),
                     "proj_err": float(f[6]), "cov_err": float(f[7]), "wall": float(f[8]), "seed": int(f[9]),
                     "raw": f})
    return rows


def _close(got, want, rel, absl=2e-9):
    return abs(got - want) <= rel * abs(want) + absl


@pytest.mark.gpu
def test_cli_eval_matches_oracle(sfdg, oracle, tmp_path):
    """generate -> sketch -> eval: the metrics row equals the oracle's exact_tail(k, Rng(seed))
    -> proj_err -> cov_err(same Rng) on the same files (sfd_main.cpp:123-143), to the 9
    decimals the CSV prints; k = 0 prints proj_err "nan" (the reference's empty optional)."""
    import paper_1602_00412_b200 as P
    mtx, sk = tmp_path / "a.mtx", tmp_path / "b.csv"
    assert run("generate", "--n", 1500, "--d", 200, "--z", 20, "--seed", 3, "--output", mtx).returncode == 0
    r = run("sketch", "--input", mtx, "--output", sk, "--ell", 20, "--seed", 4)
    assert r.returncode == 0, r.stderr
    rp, cs, vs, d = P.read_row_stream(str(mtx))
    b = np.loadtxt(sk, delimiter=",")
    for k in (5, 0):
        out = tmp_path / f"m{k}.csv"
        r = run("eval", "--matrix", mtx, "--sketch", sk, "--output", out, "--k", k, "--seed", 11)
        assert r.returncode == 0, r.stderr
        (row,) = _metrics(out)
        assert (row["algo"], row["n"], row["d"], row["ell"], row["z"], row["k"], row["seed"]) == \
            ("eval", 1500, 200, 20, 20, k, 11)
        g = oracle.rng(11)
        tail, _, _ = oracle.exact_tail(rp, cs, vs, d, k, g)
        ce = oracle.cov_err(rp, cs, vs, d, b, g, 1000)
        assert _close(row["cov_err"], ce, 1e-7)
        if k:
            pe = oracle.proj_err(rp, cs, vs, d, b, k, tail)
            assert _close(row["proj_err"], pe, 1e-7)
        else:
            assert row["raw"][6] == "nan"
    man = json.load(open(str(tmp_path / "m0.csv") + ".manifest.json"))
    assert man["command"] == "eval" and man["k"] == 0 and man["seed"] == 11 and man["sketch"] == str(sk)


@pytest.mark.gpu
def test_cli_bench_sweep_matches_oracle(sfdg, oracle, tmp_path):
    """`bench --sweep nnz --scale 0.1`: the reference's cell grid (sfd_main.cpp:157-209: scaled
    defaults, z/ell capped at d, k = max(1, min(10, ell - 1)), cell seed = seed + 1000 cell,
    fd then sfd), and every cell's metrics equal the oracle's on the same synthetic stream and
    seeds (tail_rng = seed ^ 0x5bf03635, metrics_rng = seed ^ 0x9e3779b97f4a7c15)."""
    import paper_1602_00412_b200 as P
    out = tmp_path / "bench.csv"
    r = run("bench", "--sweep", "nnz", "--scale", 0.1, "--seed", 2, "--out-csv", out)
    assert r.returncode == 0, r.stderr
    rows = _metrics(out)
    zs = [2, 3, 5, 10, 25, 50]  # max(2, llround(v * 0.1)) for v in 5, 25, 50, 100, 250, 500
    assert [x["algo"] for x in rows] == ["fd", "sfd"] * 6
    assert r.stderr.count("bench: nnz=") == 6
    for cell, z in enumerate(zs):
        seed = 2 + 1000 * cell
        for row in rows[2 * cell:2 * cell + 2]:
            assert (row["n"], row["d"], row["ell"], row["z"], row["k"], row["seed"]) == (1000, 100, 5, z, 4, seed)
            assert row["wall"] > 0
        mtx = tmp_path / f"c{cell}.mtx"
        assert run("generate", "--n", 1000, "--d", 100, "--z", z, "--seed", seed, "--output", mtx).returncode == 0
        rp, cs, vs, d = P.read_row_stream(str(mtx))
        tail, _, _ = oracle.exact_tail(rp, cs, vs, d, 4, oracle.rng(seed ^ 0x5BF03635))
        a = np.zeros((1000, d))
        for i in range(1000):
            a[i, cs[rp[i]:rp[i + 1]]] = vs[rp[i]:rp[i + 1]]
        bfd, _ = oracle.fd_sketch(a, 5)
        bsfd, _ = oracle.sketch(rp, cs, vs, d, 5, seed=seed)
        for row, b in zip(rows[2 * cell:2 * cell + 2], (bfd, bsfd)):
            pe = oracle.proj_err(rp, cs, vs, d, b, 4, tail)
            ce = oracle.cov_err(rp, cs, vs, d, b, oracle.rng(seed ^ 0x9E3779B97F4A7C15), 1000)
            assert _close(row["cov_err"], ce, 1e-6), (cell, row["algo"])
            assert pe is not None and _close(row["proj_err"], pe, 1e-6), (cell, row["algo"])
    man = json.load(open(str(out) + ".manifest.json"))
    assert man == {"command": "bench", "version": man["version"], "sweep": "nnz", "scale": 0.1, "seed": 2,
                   "fast_q": False, "out_csv": str(out)}
