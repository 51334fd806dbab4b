"""Per-source-line SASS opcode mix of an ncu capture (-lineinfo, --import-source on): for the
opcodes named (default FMUL FSEL FADD), the lines that execute most of them.

    python profiles/ncu_opmix.py gpurun_out/one_r02k_bwd.ncu-rep blend_backward [OP ...]
"""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    want = sys.argv[3:] or ["FMUL", "FSEL", "FADD"]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                          f"regex:{kern}"], capture_output=True, text=True).stdout
    header, cur, path = None, None, None
    per = defaultdict(Counter)
    tot = Counter()
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            header = r
            continue
        if header is None or r[0] == "Function Name":
            continue
        if r[0]:
            cur = f"{path}:{r[0]} {r[1].strip()[:70]}"
            continue
        ins = r[3]
        tok = ins.strip().split()
        if not tok:
            continue
        op = tok[1] if tok[0].startswith("@") else tok[0]
        op = op.split(".")[0]
        v = r[header.index("Instructions Executed", 4)]
        n = float(v) if v not in ("", "-") else 0.0
        per[op][cur] += n
        tot[op] += n
    allt = sum(tot.values())
    for op in want:
        print(f"== {op}: {100 * tot[op] / allt:.2f} % of warp instructions")
        for line, n in per[op].most_common(12):
            print(f"  {100 * n / allt:6.2f}  {line}")


if __name__ == "__main__":
    main()
