"""Attribute ncu per-SASS samples/instructions to CUDA source lines.
    python tools/sass_lines.py <cubin> <ncu --page source --csv --print-source sass> <kernel substr> <src file> [top]
The cubin is disassembled with nvdisasm --print-line-info; the kernel is the first
.text section whose name contains <kernel substr> (and 'ILb1' / 'ILb0' etc. if given)."""
import collections
import csv
import re
import subprocess
import sys

cubin, prof, kname, srcf = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
txt = subprocess.run(["/usr/local/cuda/bin/nvdisasm", "--print-line-info", cubin], capture_output=True,
                     text=True).stdout.split('\n')
start = [i for i, l in enumerate(txt) if '.section' in l and '.text.' in l and kname in l][0]
end = [i for i, l in enumerate(txt[start + 1:], start + 1) if '.section' in l]
end = end[0] if end else len(txt)
addr2line, cur = {}, None
for l in txt[start:end]:
    m = re.search(r'line (\d+)', l)
    if l.strip().startswith('//##') and m:
        f = re.search(r'File "([^"]+)"', l)
        cur = (f.group(1) if f else srcf, int(m.group(1)))
        continue
    m = re.match(r'\s*/\*([0-9a-f]+)\*/', l)
    if m and cur is not None:
        addr2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(prof)))
h = rows[1]
ai, si, ii = h.index('Address'), h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed')
samp, ins, base = collections.Counter(), collections.Counter(), None
for r in rows[2:]:
    try:
        a = int(r[ai], 16)
    except (ValueError, IndexError):
        continue
    base = a if base is None else base
    ln = addr2line.get(a - base, ('', -1))
    samp[ln] += float(r[si] or 0)
    ins[ln] += float(r[ii] or 0)
tot, toti = sum(samp.values()), sum(ins.values())
srcs = {}


def line_of(f, ln):
    if ln <= 0:
        return ''
    if f not in srcs:
        try:
            srcs[f] = open(f).read().split('\n')
        except OSError:
            srcs[f] = []
    return srcs[f][ln - 1].strip()[:90] if ln <= len(srcs[f]) else ''


print('samples', tot, 'warp instructions', toti)
for (f, ln), s_ in samp.most_common(top):
    name = f.split('/')[-1] if f else '?'
    print(f"{name[:14]:>14}:{ln:<5d} {100 * s_ / tot:5.1f}% samp {100 * ins[(f, ln)] / toti:5.1f}% ins | {line_of(f, ln)}")
