"""Summarise a torch.profiler chrome trace of bench.py --trace: per stream,
busy time and kernel families; cross-stream overlap; the per-bucket cadence
on the main stream (diagnostics for the N>1 commit pipeline)."""

import json
import re
import sys
from collections import defaultdict


def family(name):
    m = re.match(r"(?:void )?(\w+)", name)
    base = m.group(1) if m else name
    if base.startswith("fold_") and "Forest" in name:
        return base + "<Forest>"
    if base.startswith("fold_"):
        k = re.search(r"Prog\w+<?\d*>?", name)
        return base + "<" + (k.group(0) if k else "?") + ">"
    return base


def main(path):
    ev = json.load(open(path))["traceEvents"]
    ks = [e for e in ev if e.get("cat") == "kernel"]
    ks.sort(key=lambda e: e["ts"])
    t0, t1 = ks[0]["ts"], max(e["ts"] + e["dur"] for e in ks)
    span = t1 - t0
    by_stream = defaultdict(list)
    for e in ks:
        by_stream[e["args"].get("stream", e.get("tid"))].append(e)
    print("%s: %d kernels over %.0f us (4 steps)" % (path, len(ks), span))
    for s, es in sorted(by_stream.items(), key=lambda kv: -len(kv[1])):
        busy = sum(e["dur"] for e in es)
        fam = defaultdict(lambda: [0, 0.0])
        for e in es:
            f = fam[family(e["name"])]
            f[0] += 1
            f[1] += e["dur"]
        print("  stream %s: %d kernels, busy %.0f us (%.0f%%)" % (s, len(es), busy, 100 * busy / span))
        for n, (c, d) in sorted(fam.items(), key=lambda kv: -kv[1][1]):
            print("     %-48s n=%4d mean %7.1f us total %8.0f" % (n[:48], c, d / c, d))
    # union busy and pairwise overlap
    iv = sorted((e["ts"], e["ts"] + e["dur"]) for e in ks)
    union, cur = 0.0, None
    for a, b in iv:
        if cur is None or a > cur[1]:
            if cur:
                union += cur[1] - cur[0]
            cur = [a, b]
        else:
            cur[1] = max(cur[1], b)
    union += cur[1] - cur[0]
    print("  GPU busy (union) %.0f us = %.0f%% of span; idle %.0f us" % (union, 100 * union / span, span - union))
    # overlap of combine with prereduce
    comb = [(e["ts"], e["ts"] + e["dur"]) for e in ks if "Tree" in e["name"] or "combine" in e["name"]]
    pre = [(e["ts"], e["ts"] + e["dur"]) for e in ks if "Forest" in e["name"] or "ProgFull" in e["name"]]
    ov = 0.0
    for a, b in comb:
        for c, d in pre:
            ov += max(0.0, min(b, d) - max(a, c))
    tc = sum(b - a for a, b in comb)
    if tc:
        print("  combine-like %.0f us, of which %.0f us overlapped with pre-reduce-like kernels" % (tc, ov))
    # main-stream cadence: gaps between consecutive kernels on the busiest stream
    s_main = max(by_stream, key=lambda s: sum(e["dur"] for e in by_stream[s] if "barrier" in e["name"]) )
    es = by_stream[s_main]
    gaps = [es[i + 1]["ts"] - (es[i]["ts"] + es[i]["dur"]) for i in range(len(es) - 1)]
    gaps = [g for g in gaps if g >= 0]
    if gaps:
        gaps.sort()
        print("  barrier stream %s: inter-kernel gaps median %.1f us, p90 %.1f us, sum %.0f us" % (
            s_main, gaps[len(gaps) // 2], gaps[int(len(gaps) * 0.9)], sum(gaps)))




def timeline(path, start=100, count=40):
    """Print `count` kernels from index `start` in time order, both streams,
    with the host time their launch call was made (correlation id)."""
    ev = json.load(open(path))["traceEvents"]
    ks = sorted((e for e in ev if e.get("cat") == "kernel"), key=lambda e: e["ts"])
    host = {e["args"].get("correlation"): e for e in ev
            if e.get("cat") == "cuda_runtime" and "correlation" in e.get("args", {})}
    t0 = ks[start]["ts"]
    print("   gpu_start  gpu_end  stream  kernel                                   host_launch")
    for e in ks[start:start + count]:
        h = host.get(e["args"].get("correlation"))
        hl = "%8.1f" % (h["ts"] - t0) if h else "       ?"
        print("   %8.1f %8.1f  s%-4s %-40s %s" % (e["ts"] - t0, e["ts"] + e["dur"] - t0,
                                             e["args"].get("stream"), family(e["name"])[:40], hl))
    rt = defaultdict(lambda: [0, 0.0])
    for e in ev:
        if e.get("cat") == "cuda_runtime":
            rt[e["name"]][0] += 1
            rt[e["name"]][1] += e.get("dur", 0)
    print("   host runtime calls:", {k: (v[0], round(v[1] / max(1, v[0]), 1)) for k, v in rt.items()})


if __name__ == "__main__":
    if sys.argv[1] == "--timeline":
        timeline(sys.argv[2])
    else:
        for p in sys.argv[1:]:
            main(p)
