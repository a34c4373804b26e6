"""Top SASS hotspots (warp-stall samples) of an ncu report, with the CUDA line
they map to:  python tools/hotspots.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys


def main(path, top=30):
    sass = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                          capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(sass)))
    hdr = None
    out = []
    for r in rows:
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            try:
                out.append((float(d["Warp Stall Sampling (All Samples)"]), d["Address"][-5:], d["Source"][:70]))
            except ValueError:
                pass
    tot = sum(o[0] for o in out) or 1
    for v, a, s in sorted(out, reverse=True)[:top]:
        print("%6.1f%%  %s  %s" % (100 * v / tot, a, s))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
