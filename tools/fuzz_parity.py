#!/usr/bin/env python
"""fuzz_parity.py -- randomized parity sweep: the device sketcher against the CPU oracle.

Draws many small stream shapes and value/column distributions the fixed parity tests do not
cover (+-1 and integer values, head/tail and Zipf columns, duplicated rows, exact and nearly
low-rank rows, tiny d, ell = 1 and ell = d, delta / power overrides) and checks every run with
the north_star gates: B^T B within 1e-8 relative Frobenius of the oracle's, counters exact.

    python tools/fuzz_parity.py [--cases 200] [--seed 0] [--max-d 300] [--big] [--mode sfd|fd|merge]
                                [--out report.json]

Test infrastructure (uses oracle/); prints one line per failure and a JSON summary.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1602_00412_b200 as P  # noqa: E402
from oracle.oracle import Oracle, PowerConfig as OPower  # noqa: E402


def btb_rel(b1, b2):
    g1, g2 = b1.T @ b1, b2.T @ b2
    return float(np.linalg.norm(g1 - g2) / max(np.linalg.norm(g2), 1e-300))


def draw_case(g: np.random.Generator, max_d: int, big: bool = False):
    if big:  # wide sketches: ell 65..256 (trsm panels, 4-chunk SpMM, Q 3..8 verify, cluster tridiag)
        d = int(g.integers(300, max_d + 1))
        ell = int(g.integers(65, min(256, d) + 1))
        n = int(g.integers(ell, 3 * d))
        kind = str(g.choice(["gauss", "pm1", "int", "lognormal"]))
        return {"d": d, "ell": ell, "n": n, "kind": kind, "cols": str(g.choice(["uniform", "headtail", "zipf"])),
                "structure": str(g.choice(["none", "dups", "lowrank", "nearlow"])),
                "zmax": int(g.choice([3, 10, 40])), "seed": int(g.integers(0, 2**31)),
                "delta": float(g.choice([0.1, 0.01])), "q_override": int(g.choice([1, 2, 3, 4]))}
    d = int(g.choice([int(g.integers(2, 12)), int(g.integers(12, 80)), int(g.integers(80, max_d + 1))]))
    ell = int(g.choice([1, int(g.integers(1, min(d, 64) + 1)), min(d, int(g.integers(2, 9)))]))
    if g.random() < 0.05:
        ell = min(d, 64)
    n = int(g.integers(ell, 2500))
    kind = str(g.choice(["gauss", "pm1", "int", "lognormal"]))
    cols = str(g.choice(["uniform", "headtail", "zipf"]))
    structure = str(g.choice(["none", "dups", "lowrank", "nearlow"]))
    zmax = max(1, min(d, int(g.choice([2, 5, 20, d]))))
    case = {"d": d, "ell": ell, "n": n, "kind": kind, "cols": cols, "structure": structure, "zmax": zmax,
            "seed": int(g.integers(0, 2**31)), "delta": float(g.choice([0.1, 0.1, 0.01, 0.5])),
            "q_override": int(g.choice([-1, -1, -1, 1, 3, 8]))}
    return case


def make_stream(c):
    g = np.random.default_rng(c["seed"])
    d, n, zmax = c["d"], c["n"], c["zmax"]
    if c["cols"] == "zipf":
        w = 1.0 / np.arange(1, d + 1) ** 1.1
    elif c["cols"] == "headtail":
        w = np.ones(d)
        w[: max(1, d // 10)] = 20.0
    else:
        w = np.ones(d)
    w = w / w.sum()

    def value(k):
        if c["kind"] == "pm1":
            return g.choice([-1.0, 1.0], size=k)
        if c["kind"] == "int":
            return g.integers(-3, 4, size=k).astype(float)
        if c["kind"] == "lognormal":
            return g.lognormal(0.0, 2.0, size=k) * g.choice([-1.0, 1.0], size=k)
        return g.standard_normal(k)

    base = None
    if c["structure"] in ("lowrank", "nearlow"):
        r = int(g.integers(1, max(2, min(d, 2 * c["ell"] + 2))))
        base = []
        for _ in range(r):
            z = int(g.integers(1, zmax + 1))
            idx = np.sort(g.choice(d, size=z, replace=False, p=w))
            base.append((idx, value(z)))
    rows = []
    for i in range(n):
        if base is not None:
            coef = g.standard_normal(len(base))
            v = np.zeros(d)
            for (idx, val), a in zip(base, coef):
                v[idx] += a * val
            if c["structure"] == "nearlow" and g.random() < 0.3:
                j = int(g.integers(0, d))
                v[j] += 1e-7 * g.standard_normal()
            idx = np.nonzero(v)[0]
            rows.append((idx.astype(np.uint32), v[idx]))
        elif c["structure"] == "dups" and rows and g.random() < 0.5:
            rows.append(rows[int(g.integers(0, len(rows)))])
        else:
            z = int(g.integers(1, zmax + 1))
            idx = np.sort(g.choice(d, size=z, replace=False, p=w))
            vals = value(z)
            keep = vals != 0.0
            rows.append((idx[keep].astype(np.uint32), vals[keep]))
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(r[0]) for r in rows])
    cs = np.concatenate([r[0] for r in rows]) if rp[-1] else np.zeros(0, np.uint32)
    vs = np.concatenate([r[1] for r in rows]) if rp[-1] else np.zeros(0)
    return rp, cs.astype(np.uint32), vs.astype(np.float64)


def run_case(O, c):
    rp, cs, vs = make_stream(c)
    qo = None if c["q_override"] < 0 else c["q_override"]
    pw = P.PowerConfig(q_override=qo) if qo is not None else P.PowerConfig()
    opw = OPower(q_override=qo)
    res = {"case": c}
    try:
        bo, so = O.sketch(rp, cs, vs, c["d"], c["ell"], seed=c["seed"], delta=c["delta"], power=opw)
    except Exception as e:  # noqa: BLE001 -- the reference's own failure: the device must fail alike
        bo, so = None, repr(e)
    try:
        s = P.SfdSketcher(P.SketchConfig(ell=c["ell"], d=c["d"], seed=c["seed"], delta=c["delta"], power=pw))
        s.append_csr(rp, cs, vs)
        b = s.finalize()
        st = s.stats()
        s.close()
    except Exception as e:  # noqa: BLE001
        b, st = None, repr(e)
    if bo is None or b is None:
        res["ok"] = (bo is None) == (b is None)
        res["oracle"] = so if bo is None else "ok"
        res["gpu"] = st if b is None else "ok"
        return res
    res["btb"] = btb_rel(b, bo)
    res["counters"] = {k: (st[k], so[k]) for k in ("flushes", "attempts", "verifier_i", "delta_spent")}
    res["ok"] = res["btb"] <= 1e-8 and all(a == b_ for a, b_ in res["counters"].values())
    return res


def run_fd_case(O, c):
    """FdSketcher (sketch.cpp:47-78) on the same streams, densified: B^T B and shrink_count."""
    rp, cs, vs = make_stream(c)
    n, d = len(rp) - 1, c["d"]
    a = np.zeros((n, d))
    for i in range(n):
        a[i, cs[rp[i]:rp[i + 1]]] = vs[rp[i]:rp[i + 1]]
    res = {"case": c, "mode": "fd"}
    try:
        bo, co = O.fd_sketch(a, c["ell"])
    except Exception as e:  # noqa: BLE001
        bo, co = None, repr(e)
    try:
        f = P.FdSketcher(c["ell"], d)
        if c["seed"] % 2:
            f.append_csr(rp, cs, vs)
        else:
            f.append_rows(a)
        b = f.finalize()
        cg = f.shrink_count()
        f.close()
    except Exception as e:  # noqa: BLE001
        b, cg = None, repr(e)
    if bo is None or b is None:
        res["ok"] = (bo is None) == (b is None)
        res["oracle"], res["gpu"] = str(co), str(cg)
        return res
    res["btb"] = btb_rel(b, bo)
    res["counters"] = {"shrink_count": (cg, co)}
    res["ok"] = res["btb"] <= 1e-8 and cg == co
    return res


def run_merge_case(O, c):
    """merge (sketch.cpp:80-83) of two shard sketches of the stream (seeds s, s + 1)."""
    rp, cs, vs = make_stream(c)
    n = len(rp) - 1
    h = n // 2
    parts = []
    res = {"case": c, "mode": "merge"}
    for k, (r0, r1) in enumerate(((0, h), (h, n))):
        sub = (rp[r0:r1 + 1] - rp[r0], cs[rp[r0]:rp[r1]], vs[rp[r0]:rp[r1]])
        try:
            bo, _ = O.sketch(*sub, c["d"], c["ell"], seed=c["seed"] + k)
        except Exception as e:  # noqa: BLE001 -- the reference cannot sketch this shard: no merge input
            res.update({"ok": True, "skipped": repr(e)})
            return res
        parts.append(bo)
    mo = O.merge(parts[0], parts[1], c["ell"])
    mg = P.merge(parts[0], parts[1], c["ell"])
    res["btb"] = btb_rel(mg, mo)
    res["ok"] = res["btb"] <= 1e-8
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=200)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--max-d", type=int, default=300)
    ap.add_argument("--out", default="")
    ap.add_argument("--big", action="store_true", help="ell 65..256, d 300..max-d, q 1..4")
    ap.add_argument("--case", default="", help="rerun one case given as its JSON dict")
    ap.add_argument("--mode", default="sfd", choices=["sfd", "fd", "merge"],
                    help="sfd: SfdSketcher streams; fd: FdSketcher; merge: merge of two shard sketches")
    a = ap.parse_args()
    O = Oracle()
    if a.case:
        r = run_case(O, json.loads(a.case))
        print(json.dumps(r, default=str))
        return 0 if r["ok"] else 1
    g = np.random.default_rng(a.seed)
    fails, worst, t0 = [], 0.0, time.time()
    for i in range(a.cases):
        c = draw_case(g, a.max_d, a.big)
        r = {"sfd": run_case, "fd": run_fd_case, "merge": run_merge_case}[a.mode](O, c)
        worst = max(worst, r.get("btb", 0.0))
        if not r["ok"]:
            fails.append(r)
            print("FAIL", i, json.dumps(r, default=str), flush=True)
    summary = {"cases": a.cases, "failures": len(fails), "worst_btb": worst, "seconds": round(time.time() - t0, 1)}
    print(json.dumps(summary))
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"summary": summary, "failures": fails}, f, indent=1, default=str)
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
