"""Per-source-line summary of an ncu capture (needs -lineinfo builds and --import-source on):
warp-stall samples, warp-level instructions executed and the top stall reasons per CUDA line.

    python profiles/ncu_lines.py gpurun_out/one_r02bwd.ncu-rep [kernel-substring] [top]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def load(rep, kernel=None):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kernel:
        cmd += ["-k", f"regex:{kernel}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows, path, header = [], None, None
    for rec in csv.reader(io.StringIO(out)):
        if not rec:
            continue
        if rec[0] == "File Path":
            path = rec[1].split("/")[-1]
            continue
        if rec[0] == "Line No":
            header = rec
            continue
        if header is None or rec[0] in ("Function Name", "Kernel Name"):
            continue
        if rec[0]:  # a CUDA source line with its aggregated metrics
            d = dict(zip(header[2:], rec[2:]))
            d["_file"], d["_line"], d["_src"] = path, int(rec[0]), rec[1].strip()
            rows.append(d)
    return rows, header


def num(v):
    try:
        return float(v)
    except (TypeError, ValueError):
        return 0.0


def main():
    rep = sys.argv[1]
    kernel = sys.argv[2] if len(sys.argv) > 2 else None
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    rows, header = load(rep, kernel)
    stalls = [h for h in header[2:] if h.startswith("stall_") and "Not Issued" not in h]
    tot_s = sum(num(r.get("Warp Stall Sampling (All Samples)")) for r in rows) or 1.0
    tot_i = sum(num(r.get("Instructions Executed")) for r in rows) or 1.0
    agg = defaultdict(lambda: defaultdict(float))
    for r in rows:
        k = (r["_file"], r["_line"], r["_src"][:90])
        agg[k]["samples"] += num(r.get("Warp Stall Sampling (All Samples)"))
        agg[k]["inst"] += num(r.get("Instructions Executed"))
        for s in stalls:
            agg[k][s] += num(r.get(s))
    print(f"total samples {tot_s:.0f}, warp instructions {tot_i:.0f}")
    print(f"{'samp%':>6} {'inst%':>6}  file:line  top stalls  | source")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
        st = sorted(((v[s], s[6:]) for s in stalls), reverse=True)[:3]
        sts = " ".join(f"{n}:{100 * c / max(v['samples'], 1):.0f}" for c, n in st if c > 0)
        print(f"{100 * v['samples'] / tot_s:6.2f} {100 * v['inst'] / tot_i:6.2f}  {k[0]}:{k[1]}  {sts}  | {k[2]}")


if __name__ == "__main__":
    main()
