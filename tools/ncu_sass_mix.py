"""Instruction mix and stall samples by SASS opcode from an ncu source page
(run here, no GPU):

    ncu -i X.ncu-rep --page source --csv --print-source sass > x.csv
    python tools/ncu_sass_mix.py x.csv [pages [top]] > profiles/rNN_sass_mix.txt

Groups executed warp instructions by opcode (the ALU pipe takes LOP3, SHF,
PRMT, ISETP, SEL...; IMAD/IADD3 go to the FMA pipe) and reports per-page
counts when the page count of the captured launch is given."""

import collections
import csv
import sys


def main():
    path = sys.argv[1]
    pages = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    with open(path, newline="") as f:
        rows = list(csv.reader(f))
    kernel = rows[0][1] if rows and rows[0] else "?"
    hdr = rows[1]
    i_src, i_exec, i_samp = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index(
        "Warp Stall Sampling (All Samples)")
    ex, samp = collections.Counter(), collections.Counter()
    for r in rows[2:]:
        if len(r) <= i_samp or not r[i_src].strip():
            continue
        toks = r[i_src].split()
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        ex[op] += int(float(r[i_exec] or 0))
        samp[op] += int(float(r[i_samp] or 0))
    tot_e, tot_s = sum(ex.values()), sum(samp.values()) or 1
    print(f"# {kernel}")
    print(f"# {tot_e} warp instructions executed" + (f", {tot_e / pages:.1f} per page ({tot_e / pages / 2:.1f} per warp-page)" if pages else ""))
    print(f"{'opcode':10s} {'executed':>12s} {'share':>7s} {'per page':>9s} {'stall samples':>14s}")
    for op, n in ex.most_common(top or None):
        per = f"{n / pages:9.1f}" if pages else ""
        print(f"{op:10s} {n:12d} {n / tot_e:7.1%} {per} {samp[op] / tot_s:14.1%}")


if __name__ == "__main__":
    main()
