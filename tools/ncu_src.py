"""Top SASS lines by warp-stall samples for each kernel of an ncu report."""
import csv, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
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
    data = []
    for i, r in enumerate(b[2:]):
        if len(r) < len(hdr):
            continue
        try:
            data.append((int(r[iss] or 0), i, r[isrc].strip(), r[iex]))
        except ValueError:
            pass
    print('==', name[:80], 'samples', sum(d[0] for d in data))
    for d in sorted(data, reverse=True)[:top]:
        print('  %5d  #%-5d %-60s exec=%s' % d)
