"""Top SASS lines by warp-stall samples (with the dominant stall reasons) per kernel of an ncu report.
usage: python tools/ncu_src.py <report> [top] [addr_lo addr_hi]  (addresses: SASS offsets in hex)"""
import csv, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
lo = int(sys.argv[3], 16) if len(sys.argv) > 3 else None
hi = int(sys.argv[4], 16) if len(sys.argv) > 4 else None
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
blocks, cur = [], None
for r in rows:
    if r and r[0] == 'Kernel Name':
        cur = [r[1]]
        blocks.append(cur)
        continue
    if cur is not None:
        cur.append(r)
for b in blocks:
    name, hdr = b[0], b[1]
    ia, isrc = hdr.index('Address'), hdr.index('Source')
    iss, iex = hdr.index('Warp Stall Sampling (All Samples)'), hdr.index('Instructions Executed')
    reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith('stall_') and '(Not Issued)' not in h]
    data = []
    base = None
    for r in b[2:]:
        if len(r) < len(hdr):
            continue
        try:
            addr = int(r[ia], 16)
        except ValueError:
            continue
        if base is None:
            base = addr
        off = addr - base
        if lo is not None and not (lo <= off < hi):
            continue
        try:
            smp = int(r[iss] or 0)
        except ValueError:
            continue
        rs = sorted(((float(r[i] or 0), h[6:]) for i, h in reasons), reverse=True)[:3]
        data.append((smp, off, r[isrc].strip(), r[iex], rs))
    print('==', name[:80], 'samples', sum(d[0] for d in data))
    for d in sorted(data, reverse=True)[:top]:
        print('  %5d  %05x %-58s exec=%-7s %s' % (d[0], d[1], d[2][:58], d[3],
                                                  ' '.join(f'{h}={v:.0f}' for v, h in d[4] if v > 0)))
