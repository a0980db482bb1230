"""SASS evidence for the sm_100a kernels of libustfwi_b200.so: per kernel, the instruction
count and the counts of the opcodes that prove the Blackwell data movement (UTMALDG / UTMASTG
= TMA tensor load / store, UBLKCP = bulk copy, SYNCS = mbarrier, LDGSTS = cp.async) plus the
packed fp32 FADD2/FMUL2/FFMA2 and shuffles.

    python scripts/sass_summary.py [lib.so] > profiles/r2_sass_summary.txt
"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2102_00755_b200/libustfwi_b200.so"
KEYS = ["UTMALDG", "UTMASTG", "UBLKCP", "SYNCS", "LDGSTS", "FADD2", "FMUL2", "FFMA2", "SHFL", "BAR", "LDS", "STS",
        "LDG", "STG"]
out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
kern = None
stats = collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        kern = m.group(1)
        stats[kern] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]*)?", line)
    if m and kern:
        op = m.group(1)
        stats[kern]["_n"] += 1
        for k in KEYS:
            if op == k or op.startswith(k + "."):
                stats[kern][k] += 1
        if op.startswith("BAR"):
            stats[kern]["BAR"] += 0
print(f"# SASS opcode summary of {LIB} (cuobjdump -sass), sm_100a")
print("# columns: instructions " + " ".join(KEYS))
tot = collections.Counter()
for k, c in stats.items():
    dem = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
    if not any(x in dem for x in ("pencil", "zvel", "zrho", "zp", "rows", "kernel")):
        continue
    tot.update(c)
    print(f"{c['_n']:6d} " + " ".join(f"{k}={c[k]}" for k in KEYS if c[k]) + f"   {dem[:150]}")
print("# total over kernels: " + " ".join(f"{k}={tot[k]}" for k in KEYS))
