"""Summarise ncu reports into profiles/ (run here, after gpurun brought the
.ncu-rep files back): per kernel duration, DRAM bytes, FP64 pipe, occupancy;
writes profiles/traffic.json for bench.py's roofline.traffic."""
import csv, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hdr, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")].split("(")[0]}
        for w in WANT:
            if w in hdr:
                d[w] = (row[hdr.index(w)], units[hdr.index(w)])
        res.append(d)
    return res


def main():
    out_md, traffic = [], {}
    for rep, tag in [a.split(":") for a in sys.argv[1:]]:
        for d in rows(rep):
            out_md.append("| %s | %s | " % (tag, d["kernel"]) + " | ".join(
                "%s %s" % d.get(w, ("", "")) for w in WANT) + " |")
            rd = float(d["dram__bytes_read.sum"][0].replace(",", ""))
            wr = float(d["dram__bytes_write.sum"][0].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            b = rd * scale.get(d["dram__bytes_read.sum"][1], 1) + wr * scale.get(d["dram__bytes_write.sum"][1], 1)
            traffic.setdefault(tag, int(b))
    print("| tag | kernel | " + " | ".join(WANT) + " |")
    print("|" + "---|" * (len(WANT) + 2))
    print("\n".join(out_md))
    json.dump(traffic, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
