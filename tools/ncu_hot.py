"""Hot SASS instructions of an ncu --set full --import-source report (run
here, no GPU): the top instructions by warp-stall samples, each with its
dominant stall reasons and the CUDA source line it maps to.
Usage: python tools/ncu_hot.py REPORT.ncu-rep [N]"""
import csv
import io
import subprocess
import sys


def page(path, src):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', src],
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(path, n=30):
    rows = page(path, 'sass')
    hdr = rows[1]
    body = [r for r in rows[2:] if len(r) == len(hdr)]
    i_s = hdr.index('Warp Stall Sampling (All Samples)')
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith('stall_')]
    total = sum(float(r[i_s] or 0) for r in body)
    # source line per SASS address from the mixed view, when available
    line_of = {}
    mixed = page(path, 'cuda,sass')
    cur = None
    for r in mixed:
        if len(r) >= 2 and r[0].isdigit():
            cur = r[0]
        elif len(r) >= 2 and r[0].startswith('0x'):
            line_of[r[0]] = cur
    print(f'total stall samples {total:.0f}')
    ranked = sorted(enumerate(body), key=lambda x: -float(x[1][i_s] or 0))[:n]
    for idx, r in ranked:
        s = float(r[i_s] or 0)
        reasons = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
        rs = ' '.join(f'{nm}={v:.0f}' for v, nm in reasons if v > 0)
        print(f'{idx:5d} {s / total * 100:5.1f}% L{line_of.get(r[0], "?"):>5s} {r[1].strip()[:60]:60s} {rs}')


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
