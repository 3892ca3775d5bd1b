"""Per-source-line ncu warp-stall samples / executed instructions for one kernel.
usage: sass_lines.py <cubin> <mangled-substring> <ncu sass csv> [top]"""
import collections
import csv
import re
import sys

cubin_sass, fn, csvf = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
lines = open(cubin_sass).read().split('\n')
start = next(i for i, l in enumerate(lines) if l.startswith('.text.') and fn in l)
off2 = {}
cur = None
for l in lines[start + 1:]:
    if l.startswith('.text.') or l.startswith('//-----'):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m2 = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
    if m2:
        off2[int(m2.group(1), 16)] = cur
rows = list(csv.reader(open(csvf)))
h = rows[1]
i_s, i_i = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
base = int(rows[2][0], 16)
per, peri = collections.Counter(), collections.Counter()
for r in rows[2:]:
    try:
        a, s, n = int(r[0], 16), int(r[i_s] or 0), int(r[i_i] or 0)
    except ValueError:
        continue
    k = off2.get(a - base)
    per[k] += s
    peri[k] += n
tot, toti = sum(per.values()), sum(peri.values())
srcs = {}
for k, s in per.most_common(top):
    txt = ''
    if k:
        try:
            path = {'udf.cu': 'paper_2509_05595_b200/csrc/udf.cu', 'common.cuh': 'paper_2509_05595_b200/csrc/common.cuh',
                    'isect.cu': 'paper_2509_05595_b200/csrc/isect.cu', 'simplify.cu': 'paper_2509_05595_b200/csrc/simplify.cu',
                    'exact.cuh': 'paper_2509_05595_b200/csrc/exact.cuh'}.get(k[0])
            if path:
                srcs.setdefault(path, open(path).read().split('\n'))
                txt = srcs[path][k[1] - 1].strip()[:90]
        except Exception:
            pass
    print("%5.1f%% %5.1f%%  %s  %s" % (100 * s / tot, 100 * peri[k] / toti, k, txt))
