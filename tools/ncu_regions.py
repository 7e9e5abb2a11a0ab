"""Per-code-region stall samples / executed instructions of one ncu report (source page, SASS)."""
import collections, csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]; rows = r[2:]
ia = h.index('Address'); isamp = h.index('Warp Stall Sampling (All Samples)'); iex = h.index('Instructions Executed')
isrc = h.index('Source')
gran = int(sys.argv[2], 0) if len(sys.argv) > 2 else 0x800
base = int(rows[0][ia], 16)
b = collections.defaultdict(lambda: [0, 0])
ts = te = 0
for x in rows:
    a = int(x[ia], 16) - base; s = int(x[isamp] or 0); e = int(x[iex] or 0)
    b[a // gran][0] += s; b[a // gran][1] += e; ts += s; te += e
print('samples', ts, 'executed', te, 'code bytes', hex(int(rows[-1][ia], 16) - base))
for k in sorted(b):
    s, e = b[k]
    if s > ts * 0.01 or e > te * 0.01:
        print(hex(k * gran), 'samples %5.1f%%  executed %5.1f%%' % (100 * s / ts, 100 * e / te))
