"""Dump the SASS of one kernel of a library, addresses and comments stripped (for diffs):
    python tools/sass_fun.py <lib.so> '<demangled substring>' > out.txt"""
import re
import subprocess
import sys

lib, want = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for f in re.split(r"\n\s*Function : ", out)[1:]:
    name, _, body = f.partition("\n")
    dem = subprocess.run(["c++filt"], input=name.strip(), capture_output=True, text=True).stdout.strip()
    if want not in dem:
        continue
    for ln in body.splitlines():
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;?\s*(/\*.*)?$", ln)
        if m:
            print(m.group(1), m.group(2).rstrip(" ;"))
    break
