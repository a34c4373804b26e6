"""Key metrics + stall breakdown + SASS hotspots of an ncu --set full report.
    python tools/ncu_summary.py report.ncu-rep [launch_index] [top]"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum",
        "l1tex__t_bytes.sum", "sm__inst_executed.sum", "smsp__inst_executed.sum"]


def ncu_csv(args):
    return list(csv.reader(io.StringIO(subprocess.run(["ncu", *args], capture_output=True, text=True).stdout)))


def main(path, idx=0, top=25):
    rows = ncu_csv(["-i", path, "--page", "raw", "--csv"])
    hdr, units, data = rows[0], rows[1], rows[2 + idx]
    d = dict(zip(hdr, data))
    u = dict(zip(hdr, units))
    print("kernel:", d.get("Kernel Name", "")[:100])
    for k in KEYS:
        if k in d:
            print("  %-60s %s %s" % (k, d[k], u.get(k, "")))
    st = {k[len("smsp__pcsamp_warps_issue_stalled_"):]: float(d[k]) for k in hdr
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and d[k]}
    tot = sum(st.values()) or 1
    print("stalls:", ", ".join("%s %.0f%%" % (k, 100 * v / tot) for k, v in sorted(st.items(), key=lambda x: -x[1]) if v / tot > 0.02))
    src = ncu_csv(["-i", path, "--page", "source", "--csv", "--print-source", "sass"])
    h = src[1]
    out = []
    for r in src[2:]:
        if len(r) != len(h):
            continue
        e = dict(zip(h, r))
        try:
            out.append((float(e["Warp Stall Sampling (All Samples)"]), e["Address"][-5:], e["Source"].strip()[:80]))
        except ValueError:
            pass
    t = sum(o[0] for o in out) or 1
    print("hotspots:")
    for v, a, s in sorted(out, reverse=True)[:top]:
        print("  %5.1f%%  %s  %s" % (100 * v / t, a, s))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0, int(sys.argv[3]) if len(sys.argv) > 3 else 25)
