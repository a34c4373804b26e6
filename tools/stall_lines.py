"""Attribute ncu warp-stall samples to CUDA source lines.

    python tools/stall_lines.py report.ncu-rep build/obj/<file>.o <kernel-substring> [top]

ncu's CSV source export has no per-line metrics for CUDA source, so this maps
the SASS page (per-instruction samples) through nvdisasm's line table of the
same cubin (built with -lineinfo)."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def line_table(obj, kernel_sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
    cubins = [f for f in os.listdir(tmp) if f.endswith(".cubin")]
    table = {}
    for cb in cubins:
        txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cb)], capture_output=True, text=True).stdout
        cur_fn, cur_line = None, None
        for ln in txt.splitlines():
            m = re.match(r"^\.text\.(\S+):", ln)
            if m:
                cur_fn = m.group(1)
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur_line = "%s:%s" % (os.path.basename(m.group(1)), m.group(2))
                continue
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
            if m and cur_fn and kernel_sub in cur_fn:
                table[int(m.group(1), 16)] = cur_line
    return table


def main(rep, obj, kernel_sub, top=40):
    table = line_table(obj, kernel_sub)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    recs = []
    for r in rows[2:]:
        if r and r[0] == "Kernel Name" and recs:
            break  # only the first captured launch
        if len(r) == len(hdr) and r[0].startswith("0x"):
            recs.append(dict(zip(hdr, r)))
    base = int(recs[0]["Address"], 16)
    agg = collections.Counter()
    src = {}
    for r in recs:
        off = int(r["Address"], 16) - base
        line = table.get(off, "?")
        try:
            agg[line] += float(r["Warp Stall Sampling (All Samples)"])
        except ValueError:
            pass
    tot = sum(agg.values()) or 1
    files = {}
    for line, v in agg.most_common(top):
        f, _, no = line.partition(":")
        text = ""
        if f and no:
            path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1106_5694_b200", "csrc", f)
            if os.path.exists(path):
                files.setdefault(f, open(path).read().splitlines())
                text = files[f][int(no) - 1].strip()[:90]
        print("%5.1f%%  %-26s %s" % (100 * v / tot, line, text))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 40)
