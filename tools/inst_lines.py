"""Executed warp-instructions per CUDA source line of one kernel in an ncu report.
    python tools/inst_lines.py report.ncu-rep build/obj/<file>.o <mangled-kernel-substring> [top]"""
import collections, csv, io, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from stall_lines import line_table


def main(rep, obj, kern, top=30):
    table = line_table(obj, kern)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    recs = []
    for r in rows[2:]:
        if r and r[0] == "Kernel Name" and recs:
            break
        if len(r) == len(hdr) and r[0].startswith("0x"):
            recs.append(dict(zip(hdr, r)))
    base = int(recs[0]["Address"], 16)
    agg = collections.Counter()
    for r in recs:
        try:
            agg[table.get(int(r["Address"], 16) - base, "?")] += float(r["Instructions Executed"])
        except ValueError:
            pass
    tot = sum(agg.values())
    print("total warp-instructions", int(tot))
    for k, v in agg.most_common(top):
        print("%6.2f%%  %s" % (100 * v / tot, k))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 30)
