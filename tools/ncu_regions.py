"""Summarise an ncu --import-source report by SASS loop region: share of warp
stall samples, instructions, FP64 instructions and the leading stall reasons.
Usage: python tools/ncu_regions.py report.ncu-rep [--top N]"""
import csv
import io
import re
import subprocess
import sys

REASONS = ['stall_wait', 'stall_math', 'stall_not_selected', 'stall_selected', 'stall_sleep', 'stall_long_sb',
           'stall_short_sb', 'stall_dispatch', 'stall_branch_resolving', 'stall_membar', 'stall_mio', 'stall_lg',
           'stall_no_inst', 'stall_barrier', 'stall_misc']


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index('--top') + 1]) if '--top' in sys.argv else 0
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    ia, ie, isrc = col["Warp Stall Sampling (All Samples)"], col["Instructions Executed"], col["Source"]
    base = int(data[0][0], 16)
    tot = sum(int(r[ia]) for r in data)
    segs = []
    for r in data:
        m = re.search(r'BRA\s+(0x[0-9a-f]+)', r[isrc])
        if m and int(r[ie]) > 0:
            t, off = int(m.group(1), 16) - base, int(r[0], 16) - base
            if t < off:
                segs.append((t, off))

    def agg(lo, hi):
        s = {k: 0 for k in REASONS}
        n = ex = fp = 0
        for r in data:
            off = int(r[0], 16) - base
            if lo <= off <= hi:
                n += int(r[ia])
                ex += int(r[ie])
                if re.search(r'\bD(FMA|MUL|ADD)', r[isrc]):
                    fp += int(r[ie])
                for k in REASONS:
                    s[k] += int(r[col[k]])
        return n, ex, fp, s

    print(f"total samples {tot}, instructions {sum(int(r[ie]) for r in data):.4e}")
    for a, b in segs + [(0, 1 << 40)]:
        n, ex, fp, s = agg(a, b)
        if n > 0.005 * tot:
            print(f"{a:#7x}-{b:#7x} {100 * n / tot:5.1f}% samples  inst {ex:.3e}  fp64 {fp:.3e}  ",
                  {k[6:]: round(100 * v / n, 1) for k, v in s.items() if v > 0.03 * n})
    if top:
        best = sorted(data, key=lambda r: -int(r[ia]))[:top]
        for r in best:
            print(f"{int(r[0], 16) - base:#7x} {r[isrc][:56]:56s} {int(r[ia]):8d}",
                  {k[6:]: int(r[col[k]]) for k in REASONS if int(r[col[k]]) > 0.2 * int(r[ia])})


if __name__ == "__main__":
    main()
