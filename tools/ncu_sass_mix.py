"""Instruction mix and stall samples of an ncu report's SASS page, grouped by opcode, plus the
hottest contiguous regions (by executed warp instructions).  usage: ncu_sass_mix.py rep [top]"""
import csv
import subprocess
import sys
from collections import defaultdict


def load(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    # several kernels in the report: keep the LAST kernel's section (header row repeated per kernel)
    starts = [i for i, r in enumerate(rows) if 'Address' in r and 'Source' in r]
    rows = rows[starts[-1] - 1:]
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    recs = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        recs.append((int(r[ix['Address']], 16), r[ix['Source']].strip(), int(r[ix['Instructions Executed']] or 0),
                     int(r[ix['Warp Stall Sampling (All Samples)']] or 0)))
    return recs


def main(rep, top=25):
    recs = load(rep)
    base = recs[0][0]
    tot = sum(r[2] for r in recs)
    ts = sum(r[3] for r in recs)
    mix = defaultdict(lambda: [0, 0])
    for a, src, ins, smp in recs:
        op = src.split()[0] if not src.startswith('@') else src.split()[1]
        op = op.split('.')[0]
        mix[op][0] += ins
        mix[op][1] += smp
    print(f"total {tot:,} warp instr, {ts:,} stall samples")
    for op, (i, s) in sorted(mix.items(), key=lambda x: -x[1][0])[:30]:
        print(f"  {op:10s} {i/tot*100:6.2f}% instr  {s/ts*100:6.2f}% stalls")
    # regions: split at instructions whose execution count changes by > 2x
    regions = []
    cur = [recs[0]]
    for r in recs[1:]:
        p = cur[-1][2]
        if (r[2] > 2 * p + 10 or p > 2 * r[2] + 10):
            regions.append(cur)
            cur = [r]
        else:
            cur.append(r)
    regions.append(cur)
    regions.sort(key=lambda g: -sum(x[2] for x in g))
    for g in regions[:int(top)]:
        i = sum(x[2] for x in g)
        s = sum(x[3] for x in g)
        print(f"\n== region +0x{g[0][0]-base:x}..+0x{g[-1][0]-base:x}: {len(g)} instr, {i/tot*100:.2f}% executed, "
              f"{s/ts*100:.2f}% stalls, count/instr {g[0][2]}")
        for a, src, ins, smp in g[:60]:
            print(f"   +0x{a-base:05x} {ins:>11,} {smp:>6}  {src[:80]}")


if __name__ == '__main__':
    main(*sys.argv[1:])
