"""Per-source-line instruction / stall attribution of one kernel in an ncu report.

Joins ncu's per-SASS-address counts (`--page source --print-source sass`) with
the line table of the same kernel in the built library (`nvdisasm -g`, the
library is compiled with -lineinfo), then aggregates by file:line.

    python scripts/sass_lines.py gpurun_out/prof_r1f.ncu-rep k_troubled_split \
        _ZN5ucfvb16k_troubled_splitILi5ELi2ELi3ELi10ELi4EEEvNS_6LayoutENS_7PhysicsENS_7ScratchEPK7double4i
"""
import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path

LIB = Path(__file__).resolve().parents[1] / "paper_2510_25906_b200" / "lib" / "libucfvb.so"


def line_table(mangled):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", str(LIB)], cwd=d, capture_output=True, check=True)
        cub = next(p for p in Path(d).glob("solver*.cubin"))
        txt = subprocess.run(["nvdisasm", "-g", "-c", str(cub)], capture_output=True, text=True, check=True).stdout
    start = txt.index(f".text.{mangled}:")
    end = txt.find("//---------------------", start)
    cur, table = "?", {}
    for ln in txt[start:end].splitlines():
        m = re.match(r'\s*//## File "(.*)", line (\d+)', ln)
        if m:
            cur = f"{Path(m.group(1)).name}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m:
            table[int(m.group(1), 16)] = cur
    return table


def main():
    rep, kregex, mangled = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kregex}",
                          "--print-source", "sass"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    # one section per captured launch of the kernel: keep the first
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
    if len(starts) > 1:
        rows = rows[: starts[1]]
    h = next(i for i, r in enumerate(rows) if "Address" in r)
    hdr = rows[h]
    ia, ie, iw, isrc = (hdr.index("Address"), hdr.index("Instructions Executed"),
                        hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"))
    data = [r for r in rows[h + 1:] if len(r) > ie and r[ia].startswith("0x")]
    base = int(data[0][ia], 16)
    table = line_table(mangled)
    ins, stall, ops = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
    for r in data:
        off = int(r[ia], 16) - base
        key = table.get(off, "?")
        n = int(r[ie] or 0)
        w = int(r[iw] or 0)
        ins[key] += n
        stall[key] += w
        op = r[isrc].strip().split()
        op = (op[1] if op and op[0].startswith("@") and len(op) > 1 else (op[0] if op else "?")).split(".")[0]
        ops[key][op] += n
    ti, tw = sum(ins.values()) or 1, sum(stall.values()) or 1
    print(f"total warp instructions {ti}, stall samples {tw}")
    for key, n in sorted(ins.items(), key=lambda x: -x[1])[:top]:
        o = ", ".join(f"{k} {v * 100 // n}%" for k, v in ops[key].most_common(3))
        print(f"{100 * n / ti:5.1f}% ins {100 * stall[key] / tw:5.1f}% stall  {key:28s} {o}")


if __name__ == "__main__":
    main()
