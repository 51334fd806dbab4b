"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import collections
import csv
import sys


def summarise(path, skip_frames=0):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("fgs::", "").replace("<unnamed>::", "")
        agg.setdefault(name, []).append(float(d["Metric Value"]) / 1000.0)  # ns -> us
    total = sum(sum(v) for v in agg.values())
    out = []
    for k, v in agg.items():
        out.append((k, len(v), sum(v) / len(v), sum(v), 100.0 * sum(v) / total))
    return out, total


if __name__ == "__main__":
    res, total = summarise(sys.argv[1])
    print(f"{'kernel':55s} {'n':>4s} {'mean_us':>9s} {'total_us':>10s} {'share%':>7s}")
    for k, n, m, t, sh in res:
        print(f"{k:55s} {n:4d} {m:9.2f} {t:10.1f} {sh:7.2f}")
    print(f"total {total:.1f} us")


def step_share(res, names):
    """Mean-time share of each kernel within one step made of the given kernels (one launch
    each), e.g. the device-resident forward: preprocess_kernel<0>, bin_local_kernel (or bin_kernel), blend_forward."""
    pick = {}
    for k, n, m, t, sh in res:
        for want in names:
            if k.startswith(want) and want not in pick:
                pick[want] = m
    tot = sum(pick.values())
    return {k: (v, 100.0 * v / tot) for k, v in pick.items()}, tot


if __name__ == "__main__" and len(sys.argv) > 1:
    res, _ = summarise(sys.argv[1])
    for title, names in (("forward step (device-resident)", ["void preprocess_kernel<0>", "bin_local_kernel", "void bin_kernel",
                                                            "void blend_forward_kernel<0"]),
                         ("backward step", ["void blend_backward_kernel", "void preprocess_backward_kernel<0"])):
        sh, tot = step_share(res, names)
        print(f"{title}: {tot:.1f} us = " + ", ".join(f"{k.replace('void ', '')} {v:.1f} us ({p:.0f}%)"
                                                        for k, (v, p) in sh.items()))
