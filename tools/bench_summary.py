import json,sys
for line in sys.stdin:
    line=line.strip()
    if not line.startswith('{'): continue
    d=json.loads(line); r=d.get("roofline",{}); dm=d.get("dense_mask_run",{})
    print(d["config"]["workload"][:28], d["config"]["variant"], "ms=%.4f"%d["ms_per_step"], "TF=%.1f"%d["value"], r.get("bound"), "frac=%.3f"%r.get("frac",0), "tensor=%.3f"%r.get("tensor_frac",0), "dense_ms=%.3f"%dm.get("ms_per_step",0), "spd=%.2f"%dm.get("speedup_vs_dense",0), "pre_ms=%.4f"%d.get("preprocess",{}).get("ms",0))
