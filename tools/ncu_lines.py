"""Attribute ncu SASS-page stall samples / executed instructions to source lines.

usage: ncu -i rep --page source --csv --print-source=sass > sass.csv
       nvdisasm -g -c lib.cubin | (kernel section) > disasm.txt
       python tools/ncu_lines.py sass.csv disasm.txt csrc/panel1.cuh [N]
"""
import collections
import csv
import re
import sys


def main():
    sass, dis, srcf = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    line = None
    addr2line = {}
    for l in open(dis):
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            line = (m.group(1).split('/')[-1], int(m.group(2)))
            continue
        m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', l)
        if m and line:
            addr2line[int(m.group(1), 16)] = line
    rows = list(csv.reader(open(sass)))
    h = rows[1]
    idx = {k: i for i, k in enumerate(h)}
    data = [r for r in rows if len(r) == len(h) and r[0].startswith('0x')]
    base = int(data[0][0], 16)
    samp = collections.Counter()
    inst = collections.Counter()
    for r in data:
        ln = addr2line.get(int(r[0], 16) - base, ('?', 0))
        samp[ln] += int(r[idx['Warp Stall Sampling (All Samples)']] or 0)
        inst[ln] += int(r[idx['Instructions Executed']] or 0)
    tot = sum(samp.values())
    itot = sum(inst.values())
    src = open(srcf).read().split('\n')
    base_name = srcf.split('/')[-1]
    print(f"samples {tot}, warp instructions {itot}")
    for (f, l), v in samp.most_common(top):
        txt = src[l - 1].strip()[:70] if f == base_name and l > 0 else ''
        print(f"{v / tot * 100:5.1f}% smp {inst[(f, l)] / itot * 100:5.1f}% ins  {f}:{l} {txt}")


if __name__ == "__main__":
    main()
