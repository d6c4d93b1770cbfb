"""Average the per-variant TOPS of a tools/ab_w8.sh log into one table."""
import collections
import re
import sys

d = collections.defaultdict(lambda: collections.defaultdict(list))
order, cur = [], None
for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/w8ab.log"):
    if line.startswith("=="):
        cur = line.split()[1]
        if cur not in order:
            order.append(cur)
        continue
    m = re.match(r"\s+(\S+) exact=(\d) (\S+)\s+([\d.]+) ms\s+([\d.]+) TOPS", line)
    if m:
        d[(m.group(1), m.group(2), m.group(3))][cur].append(float(m.group(5)))
print(f"{'shape':34s}" + "".join(f"{v:>9s}" for v in order))
for k, per in d.items():
    print(f"{' '.join(k):34s}" + "".join(
        f"{(sum(per[v]) / len(per[v]) if per[v] else 0):9.0f}" for v in order))
