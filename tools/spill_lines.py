#!/usr/bin/env python
"""Where a kernel's local-memory spills are: STL/LDL counts per source line.
  python tools/spill_lines.py <object.o> <mangled-kernel-substring> [source.cu]"""
import collections
import os
import re
import subprocess
import sys
import tempfile

obj, pat = sys.argv[1], sys.argv[2]
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, capture_output=True)
    cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
    sass = subprocess.run(["nvdisasm", "-g", os.path.join(td, cub)], capture_output=True, text=True).stdout
lines = sass.split("\n")
starts = [i for i, l in enumerate(lines) if l.startswith(".text.") and pat in l]
src = open(sys.argv[3]).read().split("\n") if len(sys.argv) > 3 else None
for st in starts:
    end = st + 1
    while end < len(lines) and not lines[end].startswith(".text."):
        end += 1
    cur, cnt = None, collections.Counter()
    for ln in lines[st:end]:
        m = re.search(r'//## File ".*?", line (\d+)', ln)
        if m:
            cur = int(m.group(1))
            continue
        for op in ("STL", "LDL"):
            if re.search(r"\b" + op + r"\b", ln):
                cnt[(cur, op)] += 1
    print(lines[st], end - st, "lines")
    for (l, op), v in sorted(cnt.items(), key=lambda x: -x[1])[:15]:
        print(f"  {op} x{v} line {l}: {src[l - 1].strip()[:90] if src and l else ''}")
