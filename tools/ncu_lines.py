"""Map an ncu --page source --print-source sass CSV onto CUDA source lines (via nvdisasm -g of the
same object) and print the top lines by warp-stall samples and shared-memory bank-conflict excess.
usage: python tools/ncu_lines.py <src_sass.csv> <nvdisasm -g -c output> <function substring> <source.cu>"""
import collections
import csv
import re
import sys

csvp, sassp, fn, srcp = sys.argv[1:5]
rows = list(csv.reader(open(csvp)))
hdr, data = rows[1], rows[2:]
ci, si, wi = (hdr.index(k) for k in ("L1 Wavefronts Shared Excessive", "Source", "Warp Stall Sampling (All Samples)"))
lines = open(sassp).read().split("\n")
st = [i for i, l in enumerate(lines) if ".text." in l and fn in l][0]
en = next((i for i in range(st + 3, len(lines)) if "//-------------------- .text." in lines[i]), len(lines))
ln, loc = None, []
for l in lines[st:en]:
    m = re.search(r"//## File .* line (\d+)", l)
    if m:
        ln = int(m.group(1))
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(.*?);", l)
    if m:
        loc.append((ln, m.group(1)))


def op(x):
    t = x.split()
    t = t[1:] if t and t[0].startswith("@") else t
    return t[0] if t else ""


n = min(len(loc), len(data))
print("instructions", len(loc), len(data), "opcode mismatches", sum(op(loc[k][1]) != op(data[k][si]) for k in range(n)))
src = open(srcp).read().split("\n")
conf, stall = collections.Counter(), collections.Counter()
for k in range(n):
    for c, i in ((conf, ci), (stall, wi)):
        try:
            c[loc[k][0]] += int(data[k][i])
        except ValueError:
            pass
print("shared bank-conflict excess wavefronts by line")
for l, v in conf.most_common(8):
    print(f"{v:10d} {l} {src[l - 1].strip()[:100] if l else ''}")
print(f"warp-stall samples by line (total {sum(stall.values())})")
for l, v in stall.most_common(30):
    print(f"{v:10d} {l} {src[l - 1].strip()[:100] if l else ''}")
