#!/usr/bin/env python
"""Static SASS size of one kernel by source line (needs -lineinfo): python scripts/sass_lines.py <kernel-substring> [top]
Code size matters: a kernel whose hot paths do not fit the 32 KB L1.5 instruction cache pays for
every phase change with instruction-fetch stalls."""
import os, re, subprocess, sys, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(ROOT, "paper_1805_08893_b200", "libvrgeom.so")
pat = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.startswith("vr_run.")][0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", cub], cwd=d, capture_output=True, text=True).stdout
cur, key, counts, total = None, None, {}, 0
for line in dis.splitlines():
    if line.startswith("//--------------------- .text."):
        cur = line
    elif "//## File" in line:
        m = re.search(r'File "([^"]+)", line (\d+)', line)
        key = (os.path.basename(m.group(1)), int(m.group(2)))
    elif re.match(r"\s+/\*[0-9a-f]{4,}\*/", line) and cur and pat in cur:
        counts[key] = counts.get(key, 0) + 1
        total += 1
print(f"{total} SASS instructions = {total * 16 / 1024:.1f} KB")
for (f, ln), n in sorted(counts.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{n:5d}  {f}:{ln}")
