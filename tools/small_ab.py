"""A/B of the BASELINE small matrix configs (C3, C4) between two builds of
libotfx.so: python tools/small_ab.py path/to/a.so path/to/b.so [repeats]"""
import json
import os
import re
import subprocess
import sys

src = open(os.path.join(os.path.dirname(__file__), "matrix_small_timing.py")).read()
SNIP = re.search(r"SNIP = r'''(.*?)'''", src, re.S).group(1)
libs = sys.argv[1:3]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
for _ in range(reps):
    for lib in libs:
        e = dict(os.environ, OTFX_LIB=os.path.abspath(lib))
        r = subprocess.run([sys.executable, "-c", SNIP], env=e, capture_output=True, text=True,
                           timeout=300)
        print(lib, (r.stdout.strip().splitlines() or [r.stderr[-300:]])[-1], flush=True)
