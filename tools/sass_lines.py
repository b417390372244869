"""Per-source-line stall samples for one kernel of an ncu report (dev tool).

ncu's CUDA source page comes back without metrics for header-only kernels, so
this joins the SASS page (per-instruction samples) with `nvdisasm -g` line
info of the same object file by instruction offset.

usage: python tools/sass_lines.py report.ncu-rep object.o mangled_kernel_name [top]
"""
import csv
import io
import re
import subprocess
import sys
import tempfile
from collections import defaultdict
from pathlib import Path


def main() -> None:
    rep, obj, fun = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    short = re.sub(r"^_ZN4gdev\d+", "", fun)
    short = re.match(r"[A-Za-z_0-9]+?(?=E|I|N|$)", short).group(0) if short else fun
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          "regex:" + short], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    ist, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    data = [r for r in rows[2:] if len(r) > iex and r[ia].startswith("0x")]
    base = int(data[0][ia], 16)
    samples = {int(r[ia], 16) - base: (int(r[ist] or 0), int(r[iex] or 0), r[isrc].strip()) for r in data}
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", str(Path(obj).resolve())], cwd=td, check=True,
                       capture_output=True)
        cubin = next(Path(td).glob("*.cubin"))
        dis = subprocess.run(["nvdisasm", "-g", "-c", str(cubin)], capture_output=True, text=True).stdout
    # keep only the kernel's own .text section
    start = dis.index(f".text.{fun}:")
    end = dis.find(".section", start)
    dis = dis[start:end if end > 0 else len(dis)]
    line = "?"
    per_line = defaultdict(lambda: [0, 0])
    for l in dis.splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            line = f"{Path(m.group(1)).name}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m:
            off = int(m.group(1), 16)
            if off in samples:
                per_line[line][0] += samples[off][0]
                per_line[line][1] += samples[off][1]
    tot = sum(v[0] for v in per_line.values()) or 1
    for ln, (s, e) in sorted(per_line.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * s / tot:5.1f}%  {e:>11}  {ln}")


if __name__ == "__main__":
    main()
