"""Per-kernel SASS instruction histogram of the shipped library (cuobjdump -sass), the
evidence that the hot kernels are what DESIGN.md says they are: UBLKCP (bulk copy) + MUFU.EX2
+ FFMA2/FADD2 + VHMNMX (bf16x2 max) in the K3c ring kernel, UTCHMMA (tcgen05.mma) + UTMALDG
(TMA load) + LDTM (tcgen05.ld) + UTMASTG / UTMAREDG (TMA store / reduce-add) in the LM-head
GEMMs.

    python scripts/sass_histogram.py [lib] > profiles/r02_sass_histogram.txt
"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2604_26256_b200/libgrpo_async.so"
sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
demangle = lambda n: subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
funcs = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if cur and m:
        op = m.group(2) + (m.group(3) or "")
        funcs[cur][op] += 1
KEY = ("UBLKCP", "UTMALDG", "UTMASTG", "UTMAREDG", "UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "MUFU.EX2",
       "FFMA2", "FADD2", "VHMNMX", "F2FP", "DADD", "DFMA", "SYNCS", "STG", "LDS", "LDG", "BAR")
for f, c in funcs.items():
    name = demangle(f)
    if not any(k in name for k in ("stream_kernel", "rowwise_kernel", "gemm_kernel", "lmhead_kernel",
                                   "vp_kernel", "vp_stream_kernel", "bwd_kernel", "segsum", "validate")):
        continue
    tot = sum(c.values())
    keys = {k: sum(v for op, v in c.items() if op.startswith(k)) for k in KEY}
    print(f"{name}\n  {tot} instructions; " + ", ".join(f"{k} {v}" for k, v in keys.items() if v))
