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
    mhz = (d.get("clocks") or {}).get("sm_mhz")
    res[(parts[0], parts[1], parts[2])].append((d["ms_per_step"], mhz))
for k, v in sorted(res.items()):
    ms = [x for x, _ in v]
    clk = [c for _, c in v if c]
    print(k, ["%.4f" % x for x in ms], "mean %.4f" % (sum(ms) / len(ms)),
          ("MHz %s" % clk) if clk else "")
