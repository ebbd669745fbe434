#!/usr/bin/env python
"""Per-source-line executed instructions of one kernel from an ncu --set full --import-source capture.

  ncu -i rep.ncu-rep --page source --csv --print-source sass > sass.csv
  cuobjdump -xelf all libdms.so; nvdisasm -g -c dms.sm_100a.cubin > all.dis   (cut the kernel's section into gk.dis)
  python tools/ncu_source_lines.py sass.csv [top|line] [gk.dis]
The SASS rows of the ncu page are matched by offset with nvdisasm's line-info annotations."""
import csv, re, sys, collections
dis = open(sys.argv[3] if len(sys.argv) > 3 else '/tmp/w/gk.dis').read().splitlines()
line_of = {}
cur = None
inl = None
for l in dis:
    m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', l)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', l)
    if m:
        line_of[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, ii, it, isrc = hdr.index('Address'), hdr.index('Instructions Executed'), hdr.index('Thread Instructions Executed'), hdr.index('Source')
ismp = hdr.index('# Samples')
base = int(rows[2][ia], 16)
agg = collections.defaultdict(lambda: [0, 0, 0])
tot = [0, 0, 0]
for r in rows[2:]:
    off = int(r[ia], 16) - base
    k = line_of.get(off, ('?', -1))
    a = agg[k]
    a[0] += int(r[ii]); a[1] += int(r[it]); a[2] += int(r[ismp])
    tot[0] += int(r[ii]); tot[1] += int(r[it]); tot[2] += int(r[ismp])
print("total warp inst %.3f G, thread inst %.3f G, samples %d" % (tot[0] / 1e9, tot[1] / 1e9, tot[2]))
src = {}
for fn in set(k[0] for k in agg):
    try: src[fn] = open('/root/repo/paper_2206_13932_b200/csrc/' + fn).read().splitlines()
    except Exception: src[fn] = []
mode = sys.argv[2] if len(sys.argv) > 2 else 'top'
items = sorted(agg.items(), key=(lambda kv: -kv[1][0]) if mode == 'top' else (lambda kv: kv[0]))
for k, a in items[: (60 if mode == 'top' else 10000)]:
    s = src.get(k[0], [])
    text = s[k[1] - 1].strip()[:90] if 0 < k[1] <= len(s) else ''
    print("%-14s %5d  %6.2f%% winst  %6.2f%% smp  lanes %4.1f  | %s" % (k[0], k[1], 100 * a[0] / tot[0], 100 * a[2] / tot[2], a[1] / max(1, a[0]), text))
