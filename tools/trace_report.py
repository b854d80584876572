#!/usr/bin/env python
"""trace_report.py -- summarise an SFDG_TRACE timeline (JSON lines from the sketcher).

    SFDG_TRACE=/tmp/t.jsonl python -c '...sketch...'; python tools/trace_report.py /tmp/t.jsonl

Reports, over the window from the first to the last device interval: the busy fraction of
the dense-shrink chain, of verification (union over lanes; verifications are serialised),
and of the shrink phase (union over lanes), plus per-phase mean durations.
"""
import json
import sys
from collections import defaultdict


def union(iv):
    iv = sorted(iv)
    tot, cur_s, cur_e = 0.0, None, None
    for s, e in iv:
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                tot += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        tot += cur_e - cur_s
    return tot


def main(path, last=0, skip=-1):
    rows = [json.loads(l) for l in open(path) if l.strip()]
    if last:  # only the last `last` flushes (e.g. the timed step of a bench run), or `last`
        # flushes after the first `skip` ones (a bench run's timed step between warm-up and profile)
        chain = sorted((r for r in rows if r["phase"] == "dense_shrink"), key=lambda r: r["gpu_end_us"])
        chain = chain[-last:] if skip < 0 else chain[skip:skip + last]
        t_lo = min(r["gpu_start_us"] for r in chain)
        t_hi = max(r["gpu_end_us"] for r in chain)
        # the same flush ids recur across sketcher resets: keep intervals inside the step
        rows = [dict(r, gpu_start_us=max(r["gpu_start_us"], t_lo), gpu_end_us=min(r["gpu_end_us"], t_hi))
                for r in rows if r["gpu_end_us"] > t_lo and r["gpu_start_us"] < t_hi]  # clipped to the step
    by = defaultdict(list)
    for r in rows:
        by[r["phase"]].append((r["gpu_start_us"], r["gpu_end_us"]))
    t0 = min(s for v in by.values() for s, _ in v)
    t1 = max(e for v in by.values() for _, e in v)
    span = t1 - t0
    print(f"window {span / 1e3:.1f} ms, {len(by.get('dense_shrink', []))} chain steps")
    for ph in sorted(by):
        iv = by[ph]
        d = [e - s for s, e in iv]
        print(f"{ph:13s} n={len(iv):5d} mean {sum(d) / len(d):8.1f} us  sum {sum(d) / 1e3:8.1f} ms  "
              f"union busy {100 * union(iv) / span:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0, int(sys.argv[3]) if len(sys.argv) > 3 else -1)
