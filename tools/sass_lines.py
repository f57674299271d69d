#!/usr/bin/env python
"""Per-source-line attribution of an ncu SASS page (measurement aid).

Joins ncu's per-instruction SASS page (`ncu -i X.ncu-rep --page source --csv
--print-source sass`) with the line table of the same cubin
(`nvdisasm -g`) by instruction offset, and prints the source lines with the
most warp-stall samples (where the kernel's time goes) and executed
instructions.

    python tools/sass_lines.py --cubin trace_fp64.sm_100a.cubin \
        --kernel trace_pool_fp64_lean_mgILi7ELb0ELb1E --sass mg_sass.csv [--top 40]

The cubin comes from the library that ran under ncu:
`cuobjdump -xelf trace_fp64.sm_100a.cubin paper_1810_00188_b200/libermc_b200.so`.
"""
from __future__ import annotations

import argparse
import csv
import re
import subprocess
from collections import defaultdict
from pathlib import Path


def line_table(cubin, kernel):
    dis = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True,
                         check=True).stdout.splitlines()
    sec = re.compile(r"^\s*\.section\s+\.text\.(\S+?),")
    loc = re.compile(r'//## File "([^"]+)", line (\d+)')
    ins = re.compile(r"/\*([0-9a-f]{4,})\*/")
    table, cur, inside = {}, None, False
    for ln in dis:
        m = sec.match(ln)
        if m:
            inside = kernel in m.group(1)
            cur = None
            continue
        if not inside:
            continue
        m = loc.search(ln)
        if m:
            cur = (Path(m.group(1)).name, int(m.group(2)))
            continue
        m = ins.search(ln)
        if m and cur:
            table[int(m.group(1), 16)] = cur
    return table


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cubin", required=True)
    ap.add_argument("--kernel", required=True, help="substring of the mangled kernel name")
    ap.add_argument("--sass", required=True, help="ncu --page source --print-source sass csv")
    ap.add_argument("--src-root", default=str(Path(__file__).resolve().parent.parent /
                                              "paper_1810_00188_b200" / "csrc"))
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    table = line_table(a.cubin, a.kernel)
    rows = list(csv.reader(open(a.sass)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    col = {k: hdr.index(k) for k in ("Address", "Warp Stall Sampling (All Samples)",
                                     "Instructions Executed",
                                     "Thread Instructions Executed")}
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    body = [r for r in rows[hdr_i + 1:] if r and r[0].startswith("0x")]
    base = int(body[0][col["Address"]], 16)
    agg = defaultdict(lambda: [0, 0, 0, defaultdict(int)])
    tot = [0, 0, 0]
    miss = 0
    for r in body:
        off = int(r[col["Address"]], 16) - base
        key = table.get(off)
        if key is None:
            miss += 1
            key = ("?", 0)
        s = int(r[col["Warp Stall Sampling (All Samples)"]] or 0)
        wi = int(r[col["Instructions Executed"]] or 0)
        ti = int(r[col["Thread Instructions Executed"]] or 0)
        e = agg[key]
        e[0] += s
        e[1] += wi
        e[2] += ti
        for i in stall_cols:
            v = int(r[i] or 0)
            if v:
                e[3][hdr[i][6:]] += v
        tot[0] += s
        tot[1] += wi
        tot[2] += ti
    src = {}
    for f in {k[0] for k in agg}:
        p = Path(a.src_root) / f
        if p.exists():
            src[f] = p.read_text().splitlines()
    print(f"instructions {len(body)}, unmapped {miss}; samples {tot[0]}, warp inst {tot[1]}, "
          f"thread inst {tot[2]}")
    print(f"{'samples%':>8} {'inst%':>6}  line  top stalls | source")
    for key, e in sorted(agg.items(), key=lambda kv: -kv[1][0])[:a.top]:
        f, ln = key
        text = src.get(f, [])[ln - 1].strip() if f in src and 0 < ln <= len(src[f]) else ""
        stalls = ", ".join(f"{k} {v * 100 // max(e[0], 1)}%" for k, v in
                           sorted(e[3].items(), key=lambda kv: -kv[1])[:2])
        print(f"{100 * e[0] / max(tot[0], 1):8.2f} {100 * e[1] / max(tot[1], 1):6.2f}  "
              f"{f}:{ln}  [{stalls}] | {text[:90]}")


if __name__ == "__main__":
    main()
