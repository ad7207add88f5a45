"""Summarise ncu captures / launch lists into the markdown tables kept under profiles/.

    python profiles/summarize.py raw   <report.ncu-rep | raw.csv>   > profiles/<name>.md
    python profiles/summarize.py launches <launches.csv>  > profiles/<name>.md
"""

from __future__ import annotations

import collections
import csv
import io
import re
import subprocess
import sys

RAW_KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def short(name: str) -> str:
    n = name.split("(")[0].replace("void ", "")
    return re.sub(r"^kvt::", "", n)


def raw(path: str) -> None:
    if path.endswith(".csv"):  # exported on the GPU box with `ncu -i … --page raw --csv`
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    out = out[out.index('"ID"'):]
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"ncu --set full summary of `{path}` (cold-cache, serialised replay; one launch per kernel)\n")
    cols = [k for k, _ in RAW_KEYS if k in hdr]
    print("| kernel | " + " | ".join(lbl for k, lbl in RAW_KEYS if k in hdr) + " |")
    print("|---" * (len(cols) + 1) + "|")
    for r in rows[2:]:
        vals = []
        for k in cols:
            v, u = r[hdr.index(k)], units[hdr.index(k)]
            vals.append(f"{v} {u}".strip())
        print(f"| {short(r[hdr.index('Kernel Name')])} | " + " | ".join(vals) + " |")
    stall = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    print("\nTop warp-stall samples per kernel:\n")
    for r in rows[2:]:
        pairs = []
        for h in stall:
            try:
                pairs.append((float(r[hdr.index(h)].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
        pairs.sort(reverse=True)
        tot = sum(p for p, _ in pairs) or 1.0
        print(f"* {short(r[hdr.index('Kernel Name')])}: " + ", ".join(f"{n} {100 * p / tot:.0f}%" for p, n in pairs[:4]))


def launches(path: str) -> None:
    import gzip
    fh = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
    rows = [r for r in csv.reader(fh) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        k = short(r[ki])
        tot[k] += v
        cnt[k] += 1
    mine = {k: v for k, v in tot.items() if not k.startswith("at::") and "elementwise" not in k and "enable_if" not in k}
    allk = sum(mine.values()) or 1.0
    print(f"Launch list `{path}` (ncu gpu__time_duration.sum, --clock-control none; cold, serialised)\n")
    print("| kernel | launches | total us | avg us | share of our kernels |")
    print("|---|---|---|---|---|")
    for k, v in sorted(mine.items(), key=lambda x: -x[1]):
        print(f"| {k} | {cnt[k]} | {v / 1e3:.1f} | {v / cnt[k] / 1e3:.2f} | {100 * v / allk:.1f}% |")


def traffic(spec: str) -> None:
    """traffic <workload>=<raw.csv>[,<workload>=<raw.csv>...] -> JSON on stdout: per bench stage, the
    DRAM bytes (read + write) of the first captured launch of its kernel (a layer >= 2 launch)."""
    import json
    out = {}
    for item in spec.split(","):
        wl, path = item.split("=")
        txt = open(path).read()
        rows = list(csv.reader(io.StringIO(txt[txt.index('"ID"'):])))
        hdr, units = rows[0], rows[1]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        stages = {}
        for r in rows[2:]:
            name = short(r[hdr.index("Kernel Name")])
            stage = next((st for key, st in (("score", "score"), ("attn", "attn"), ("bounds", "bounds"),
                                              ("select", "select"), ("plan", "plan")) if key in name), None)
            if stage is None or stage in stages:
                continue
            b = sum(float(r[hdr.index(m)].replace(",", "")) * scale[units[hdr.index(m)]]
                    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            stages[stage] = {"kernel": name, "dram_bytes": b, "layer": 2}
        out[wl] = stages
    print(json.dumps({"source": "ncu --set full, one layer-2 launch per kernel (tools/gpu_prof.sh)", "workloads": out},
                     indent=1))


if __name__ == "__main__":
    {"raw": raw, "launches": launches, "traffic": traffic}[sys.argv[1]](sys.argv[2])
