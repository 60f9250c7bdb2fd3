"""Map an ncu SASS source-page CSV (ncu -i rep --page source --csv --print-source sass)
onto CUDA source lines via nvdisasm --print-line-info of the same cubin.
usage: sass_lines.py page.csv all.sass kernel_substring source.cu items [top]"""
import collections
import csv
import re
import sys

page, sass, kname, srcf, items = sys.argv[1:6]
top = int(sys.argv[6]) if len(sys.argv) > 6 else 30
items = float(items)
txt = open(sass).read().split('\n')
start = [i for i, l in enumerate(txt) if l.startswith('.text.') and kname in l][0]
line, off2line = None, {}
base = srcf.split('/')[-1]
for l in txt[start + 1:]:
    if l.startswith('//---------------------'):
        break
    m = re.search(r'line (\d+)', l)
    if '//## File' in l and m:
        line = int(m.group(1)) if base in l else -int(m.group(1))
        continue
    m2 = re.search(r'/\*([0-9a-f]{4})\*/\s+\S', l)
    if m2:
        off2line[int(m2.group(1), 16)] = line
rows = list(csv.reader(open(page)))
h, data = rows[1], rows[2:]
ie, si = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
sc = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
b0 = int(data[0][0], 16)
agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
for r in data:
    a = agg[off2line.get(int(r[0], 16) - b0)]
    a[0] += float(r[ie] or 0)
    a[1] += float(r[si] or 0)
    for i in sc:
        try:
            a[2][h[i]] += float(r[i] or 0)
        except ValueError:
            pass
print("instr/item", sum(a[0] for a in agg.values()) / items, "samples", sum(a[1] for a in agg.values()))
src = open(srcf).read().split('\n')
for ln, (ins, smp, st) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    s = src[ln - 1].strip()[:70] if ln and ln > 0 else f'(other {ln})'
    print(f"{ins / items:7.1f} {smp:8.0f} {[(k[6:], int(v)) for k, v in st.most_common(2)]} L{ln}: {s}")
