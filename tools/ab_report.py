"""Summarise gpurun_out/ab.log (tools/ab.sh) per config and library."""
import collections
import json

res = collections.defaultdict(list)
for line in open("gpurun_out/ab.log"):
    parts = line.split(" ", 3)
    try:
        d = json.loads(parts[3])
    except Exception:
        continue
    res[(parts[0], parts[1], parts[2])].append(d["ms_per_step"])
for k, v in sorted(res.items()):
    print(k, ["%.4f" % x for x in v], "mean %.4f" % (sum(v) / len(v)))
