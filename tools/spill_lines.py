"""Source lines of local-memory spills (STL/LDL) in one kernel of a cubin disassembly.

    cuobjdump -xelf all build/obj/attn_fwd.o; nvdisasm -g -c attn_fwd.sm_100a.cubin > all.dis
    python tools/spill_lines.py all.dis <mangled-name-substring>
"""
import re
import sys

path, fun = sys.argv[1], sys.argv[2]
inside, cur, hits = False, None, {}
for line in open(path):
    if line.startswith("//--------------------- .text."):
        inside = fun in line
        continue
    if not inside:
        continue
    m = re.search(r'line (\d+)', line) if line.lstrip().startswith("//##") else None
    if m:
        cur = int(m.group(1))
        continue
    if re.search(r"\b(STL|LDL)(\.[A-Z0-9]+)*\s", line):
        hits[cur] = hits.get(cur, 0) + 1
for k in sorted(hits, key=lambda x: x or 0):
    print(k, hits[k])
