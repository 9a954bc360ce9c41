"""Stall samples (all / long-scoreboard) and executed instructions per CUDA source line of an
ncu report (ncu --page source --print-source cuda,sass), the top lines printed."""
import csv
import subprocess
import sys


def main(rep, top=45):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout
    cur = None
    hdr = None
    recs = []
    for r in csv.reader(out.splitlines()):
        if len(r) == 2 and r[0] == 'File Path':
            cur = r[1].split('/')[-1]
            continue
        if r and r[0] == 'Line No':
            hdr = r
            ix = {}
            for i, h in enumerate(hdr):
                ix.setdefault(h, i)
            lsb = [i for i, h in enumerate(hdr) if h == 'stall_long_sb']
            continue
        if hdr and len(r) == len(hdr) and r[0] not in ('', '-'):
            try:
                s = int(r[ix['Warp Stall Sampling (All Samples)']] or 0)
                ins = int(r[ix['Instructions Executed']] or 0)
                ls = int(r[lsb[0]] or 0) if lsb else 0
            except ValueError:
                continue
            recs.append((cur, int(r[0]), s, ins, ls, r[1].strip()))
    ts = sum(x[2] for x in recs) or 1
    ti = sum(x[3] for x in recs) or 1
    tl = sum(x[4] for x in recs) or 1
    print(f"stall samples {ts:,}  warp instructions {ti:,}  long-scoreboard samples {tl:,}")
    for x in sorted(recs, key=lambda x: -x[2])[:top]:
        print(f"{x[0]}:{x[1]} stall {x[2] / ts * 100:5.2f}% lsb {x[4] / ts * 100:5.2f}% inst {x[3] / ti * 100:5.2f}%  {x[5][:80]}")


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 45)
