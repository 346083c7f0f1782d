"""Attribute ncu source-page samples of the decompile kernel to source lines.

    python tools/ncu_source_lines.py <source.csv[.gz]> <libupy_cuda.so the profile ran> [kernel substring]

`ncu --page source --csv` only lists SASS; this maps each SASS address to the
file:line nvdisasm -g reports for the profiled library (built with -lineinfo),
then prints stall samples, executed instructions and local-memory (LDL/STL)
instructions per source line and per file.
"""
import collections
import csv
import gzip
import os
import re
import subprocess
import sys
import tempfile


def line_map(so_path, kernel="decompile"):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so_path)], cwd=tmp, check=True,
                   stdout=subprocess.DEVNULL)
    amap = {}
    for cub in sorted(f for f in os.listdir(tmp) if f.endswith(".cubin")):
        txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True,
                             text=True).stdout
        sec = cur = None
        for line in txt.splitlines():
            if line.lstrip().startswith(".section"):
                sec = line.split()[1].strip(",")
            m = re.search(r'//## File "([^"]+)", line (\d+)', line)
            if m:
                cur = (m.group(1).split("/")[-1], int(m.group(2)))
                continue
            m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
            if m and sec and kernel in sec:
                amap[int(m.group(1), 16)] = cur
    return amap


def main(src_csv, so_path, kernel="decompile"):
    amap = line_map(so_path, kernel)
    opener = gzip.open if src_csv.endswith(".gz") else open
    rows = csv.reader(opener(src_csv, "rt"))
    next(rows)
    hdr = next(rows)
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iss, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    base = None
    by_line = collections.defaultdict(lambda: [0, 0, 0, 0])
    tot = [0, 0]
    for r in rows:
        if len(r) <= iex:
            continue
        a = int(r[ia], 16)
        base = a if base is None else base
        src = r[isrc].split()
        op = (src[1] if src and src[0].startswith("@") and len(src) > 1 else (src[0] if src else ""))
        s, ex = int(r[iss]), int(r[iex])
        L = by_line[amap.get(a - base, ("?", 0))]
        L[0] += s
        L[1] += ex
        if op.startswith("LDL"):
            L[2] += ex
        if op.startswith("STL"):
            L[3] += ex
        tot[0] += s
        tot[1] += ex
    print("total stall samples", tot[0], "warp instructions", tot[1])
    print("--- top source lines by stall samples")
    for k, v in sorted(by_line.items(), key=lambda kv: -kv[1][0])[:45]:
        print(f"{k[0]:16s}:{k[1]:5d} samples {v[0]:8d} ({100 * v[0] / tot[0]:5.2f}%) inst {v[1]:11d} "
              f"LDL {v[2]:10d} STL {v[3]:10d}")
    by_file = collections.defaultdict(lambda: [0, 0, 0, 0])
    for k, v in by_line.items():
        f = by_file[k[0]]
        for i in range(4):
            f[i] += v[i]
    print("--- by file")
    for k, v in sorted(by_file.items(), key=lambda kv: -kv[1][0]):
        print(f"{k:18s} samples {100 * v[0] / tot[0]:6.2f}%  inst {v[1]:11d} LDL {v[2]:10d} STL {v[3]:10d}")


if __name__ == "__main__":
    main(*sys.argv[1:4])
