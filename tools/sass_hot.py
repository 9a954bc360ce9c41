"""Hot SASS regions of an ncu report: instructions executed and stall samples per
instruction, grouped into runs, printed with the top instructions (ncu --page source)."""
import csv
import subprocess
import sys


def main(rep, top=60):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = rows[2:]
    tot_inst = sum(int(r[ix['Instructions Executed']] or 0) for r in data if len(r) == len(hdr))
    tot_samp = sum(int(r[ix['Warp Stall Sampling (All Samples)']] or 0) for r in data if len(r) == len(hdr))
    print(f"total warp instructions {tot_inst:,}  stall samples {tot_samp:,}")
    recs = []
    for i, r in enumerate(data):
        if len(r) != len(hdr):
            continue
        recs.append((i, r[ix['Source']].strip(), int(r[ix['Instructions Executed']] or 0),
                     int(r[ix['Warp Stall Sampling (All Samples)']] or 0)))
    # print in address order, only instructions with significant share
    for i, src, ins, smp in recs:
        if ins > tot_inst * 0.002 or smp > tot_samp * 0.004:
            print(f"{i:5d} {ins/ max(1,tot_inst)*100:6.2f}% {smp/max(1,tot_samp)*100:6.2f}%  {src[:90]}")


if __name__ == '__main__':
    main(sys.argv[1])


def blocks(rep, width=40):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    tot_inst = sum(int(r[ix['Instructions Executed']] or 0) for r in data)
    tot_samp = sum(int(r[ix['Warp Stall Sampling (All Samples)']] or 0) for r in data)
    for b0 in range(0, len(data), width):
        blk = data[b0:b0 + width]
        ins = sum(int(r[ix['Instructions Executed']] or 0) for r in blk)
        smp = sum(int(r[ix['Warp Stall Sampling (All Samples)']] or 0) for r in blk)
        if ins > 0.01 * tot_inst or smp > 0.01 * tot_samp:
            ops = {}
            for r in blk:
                op = r[ix['Source']].strip().split()[0] if r[ix['Source']].strip() else ''
                if op.startswith('@'):
                    op = r[ix['Source']].strip().split()[1]
                ops[op.split('.')[0]] = ops.get(op.split('.')[0], 0) + int(r[ix['Instructions Executed']] or 0)
            top = sorted(ops.items(), key=lambda x: -x[1])[:5]
            print(f"[{b0:5d}-{b0+width:5d}] inst {ins/tot_inst*100:6.2f}%  stalls {smp/tot_samp*100:6.2f}%  "
                  + ' '.join(f"{k}:{v/max(1,ins)*100:.0f}%" for k, v in top))
