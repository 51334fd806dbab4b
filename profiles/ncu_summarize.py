"""Summarise an `ncu --set full` report of one forward+backward (profiles/ncu_driver.py) per
kernel, and write profiles/ncu_traffic.json: DRAM bytes (read + write) per launch of each
bench stage, which bench.py reports as roofline.traffic.

    python profiles/ncu_summarize.py gpurun_out/full.ncu-rep profiles/r01_ncu_full.md
"""
import csv
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__bytes.sum.per_second", "dram_bw"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
]

# bench.py stage -> kernels it times
STAGES = {
    "preprocess": ["preprocess_kernel"],
    "binning+sort": ["bin_"],
    "raster": ["blend_forward_kernel"],
    "raster_backward": ["blend_backward_kernel"],
    "preprocess_backward": ["preprocess_backward_kernel"],
}


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return float(v) * scale


def to_us(v, unit):
    return float(v) * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "second": 1e6}.get(unit, 1)


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        d = {"kernel": name.replace("void ", "").replace("fgs::", "").replace("(anonymous namespace)::", "")
             .replace("<unnamed>::", "").replace("unnamed>::", "")}
        for m, key in METRICS:
            if m not in hdr:
                continue
            i = hdr.index(m)
            v = r[i].replace(",", "")
            if key == "time":
                d[key] = to_us(v, units[i])
            elif key in ("dram_read", "dram_write"):
                d[key] = to_bytes(v, units[i])
            elif key == "dram_bw":
                d[key] = to_bytes(v, units[i].replace("/second", "").replace("/s", "")) / 1e9  # GB/s
            else:
                try:
                    d[key] = float(v)
                except ValueError:
                    d[key] = v
        res.append(d)
    return res


def main(rep, md_out):
    ks = load(rep)
    lines = [f"# ncu --set full summary ({os.path.basename(rep)})", "",
             "Cold-cache, serialised replay (ncu); use for traffic and the kernel mix, not absolute speed.", "",
             "| kernel | us | DRAM read MB | DRAM write MB | DRAM GB/s | SM %peak | issue % | occupancy % | regs | grid x block |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    for d in ks:
        lines.append(f"| {d['kernel']} | {d.get('time', 0):.1f} | {d.get('dram_read', 0) / 1e6:.1f} | "
                     f"{d.get('dram_write', 0) / 1e6:.1f} | {d.get('dram_bw', 0):.0f} | {d.get('sm_%peak', 0):.1f} | "
                     f"{d.get('issue_%', 0):.1f} | {d.get('occupancy_%', 0):.1f} | {d.get('regs', 0):.0f} | "
                     f"{d.get('grid', 0):.0f} x {d.get('block', 0):.0f} |")
    traffic = {}
    for stage, names in STAGES.items():
        tot, seen = 0.0, 0
        for n in names:
            for d in ks:
                if d["kernel"].startswith(n):
                    tot += d.get("dram_read", 0) + d.get("dram_write", 0)
                    seen += 1
                    break
        if seen == len(names):
            traffic[stage] = int(tot)
    lines += ["", "DRAM bytes per launch by bench stage (profiles/ncu_traffic.json):", "", "```",
              json.dumps(traffic, indent=1), "```", ""]
    with open(md_out, "w") as f:
        f.write("\n".join(lines))
    with open(os.path.join(HERE, "ncu_traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
