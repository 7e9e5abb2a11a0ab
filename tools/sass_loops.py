"""List the innermost SASS loops that contain FP math (size / instruction mix), from cuobjdump -sass output."""
import collections, re, sys
ins = []
for l in open(sys.argv[1]).read().splitlines():
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2)))
addr = {a: i for i, (a, _) in enumerate(ins)}
back = []
for i, (a, t) in enumerate(ins):
    if 'BRA' in t:
        m = re.search(r'0x([0-9a-f]+)', t)
        if m and int(m.group(1), 16) < a and int(m.group(1), 16) in addr:
            back.append((addr[int(m.group(1), 16)], i))
res = []
for s, e in back:
    c = collections.Counter(re.sub(r'^@!?U?P\w+\s+', '', x).split()[0].split('.')[0] for _, x in ins[s:e + 1])
    if c['FFMA'] + c['FADD'] + c['DFMA'] > 0:
        res.append((e - s + 1, s, c))
print('total instructions', len(ins))
for n, s, c in sorted(res)[:int(sys.argv[2]) if len(sys.argv) > 2 else 6]:
    print(hex(ins[s][0]), 'len', n, 'bytes', 16 * n, {k: c[k] for k in ('FFMA', 'FMUL', 'FADD', 'SHFL', 'LDS', 'STG', 'IMAD', 'ISETP', 'BRA', 'BSSY', 'FSEL', 'SEL')})
