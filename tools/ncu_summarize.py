"""Summarise ncu output for profiles/.

  python tools/ncu_summarize.py launches LAUNCHES.csv > profiles/rX/launch_list_summary.txt
  python tools/ncu_summarize.py full REPORT.ncu-rep > profiles/rX/ncu_full_<kernel>.txt

`launches` groups a `--metrics gpu__time_duration.sum --csv` launch list by
kernel (count, total us, share of GPU time); `full` prints the details page of
a `--set full` capture (section | metric | unit | value) plus the DRAM bytes
the roofline's `traffic` field quotes.  Run here, on the files gpurun brought
back; needs the ncu CLI only for `full`.
"""

import csv
import io
import subprocess
import sys
from collections import OrderedDict


def _rows(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    return list(csv.DictReader(io.StringIO("".join(lines))))


def launches(path):
    agg = OrderedDict()
    for r in _rows(path):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1000.0 if unit == "ns" else (v * 1000.0 if unit == "ms" else v)
        k = r["Kernel Name"]
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + us)
    total = sum(t for _, t in agg.values()) or 1.0
    print("# kernel | launches | total us | share of GPU time (ncu: cold-cache, serialised)")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print("%s | %d | %.1f | %.1f%%" % (k[:110], n, t, 100.0 * t / total))


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"],
                         check=True, capture_output=True, text=True).stdout
    rows = list(csv.DictReader(io.StringIO(out)))
    if not rows:
        print("# empty report")
        return
    print("# kernel: %s  grid %s block %s" % (rows[0]["Kernel Name"], rows[0]["Grid Size"],
                                                 rows[0]["Block Size"]))
    for r in rows:
        if r.get("Metric Name"):
            print("%s | %s | %s | %s" % (r["Section Name"], r["Metric Name"], r["Metric Unit"],
                                         r["Metric Value"]))
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"],
                         check=True, capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) >= 3:
        head, units, vals = rr[0], rr[1], rr[2]
        for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                     "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                     "dram__throughput.avg.pct_of_peak_sustained_elapsed"):
            if name in head:
                i = head.index(name)
                print("raw | %s | %s | %s" % (name, units[i], vals[i]))


_UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def traffic(path, out="profiles/ncu_traffic.json", source=None):
    """Merge the per-launch DRAM bytes of every kernel in a --set full report
    into profiles/ncu_traffic.json (read by bench.py's roofline.traffic)."""
    import json
    import re
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"],
                         check=True, capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    head, units = rr[0], rr[1]
    try:
        with open(out) as f:
            doc = json.load(f)
    except (OSError, ValueError):
        doc = {"kernels": {}}
    for vals in rr[2:]:
        name = vals[head.index("Kernel Name")]
        # template arguments as the bench names them: drop the `void ` and
        # the parameter list
        key = re.sub(r"^void ", "", name)
        key = re.sub(r"\((FoldParams|BarrierParams)\)$", "", key).replace(" >", ">")
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = head.index(m)
            b += float(vals[i].replace(",", "")) * _UNIT.get(units[i], 1.0)
        t = head.index("gpu__time_duration.sum")
        doc["kernels"][key] = {"dram_bytes": b, "duration": vals[t], "duration_unit": units[t],
                               "report": source or path}
    with open(out, "w") as f:
        json.dump(doc, f, indent=1, sort_keys=True)
    print(json.dumps(doc["kernels"], indent=1))


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic}[sys.argv[1]](*sys.argv[2:])
