"""Dump (or count) the SASS of one kernel of a built library:
  python tools/sass.py REGEX [LIB] [--count]   (cuobjdump -sass, no GPU needed)"""
import re
import subprocess
import sys

pat = re.compile(sys.argv[1])
lib = next((a for a in sys.argv[2:] if not a.startswith("--")), "paper_2505_13215_b200/libhgs_gpu.so")
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
cur, body = None, {}
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        body[cur] = []
    elif cur and re.match(r"\s+/\*[0-9a-f]{4,6}\*/", line):
        body[cur].append(line.split(";")[0].split("*/", 1)[1].strip())
for name, ins in body.items():
    if pat.search(name):
        print(f"== {name}: {len(ins)} instructions")
        if "--count" not in sys.argv:
            for i, s in enumerate(ins):
                print(f"{i:5d} {s}")
