"""Merge the per-rank torch.profiler traces of `bench.py --trace` on one time
axis (the traces' timestamps are host-clock microseconds, comparable across
the ranks of one box) and print a window of kernels from every rank: who
starts and ends what when (diagnostics for the N>1 commit pipeline)."""

import json
import sys

from trace_summary import family

SHORT = {"fold_direct_pair_kernel": "COMB", "barrier_kernel": "BAR"}


def label(name):
    f = family(name)
    base = f.split("<")[0]
    if base in SHORT:
        return SHORT[base]
    if "ProgFull<0>" in f:
        return "copy"
    if "ProgFixed" in f:
        return "COMB-fixed"
    if "Forest" in f or "ProgFull<3>" in f or "ProgFull<4>" in f:
        return "pre"
    return f[:18]


def main(paths, start_frac=0.5, count=60):
    ks = []
    for r, p in enumerate(paths):
        ev = json.load(open(p))["traceEvents"]
        ks += [(e["ts"], e["ts"] + e["dur"], r, "%s s%s" % (label(e["name"]), e["args"].get("stream")))
               for e in ev if e.get("cat") == "kernel"]
    ks.sort()
    i0 = int(len(ks) * start_frac)
    t0 = ks[i0][0]
    print("  start     end   dur  rank kernel")
    for a, z, r, n in ks[i0:i0 + count]:
        print("%7.1f %7.1f %5.1f  r%d   %s%s" % (a - t0, z - t0, z - a, r, "    " * r, n))


if __name__ == "__main__":
    main(sys.argv[1:])
