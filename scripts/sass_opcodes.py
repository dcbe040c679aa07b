"""Per-kernel SASS opcode summary of the product library (cuobjdump -sass):
the instructions that prove which hardware paths a kernel uses -- bulk copies
(UBLKCP), TMA (UTMALDG / UTMASTG), mbarrier / async-transaction syncs (SYNCS),
DSMEM cluster accesses and barriers, fp64 tensor-core MMA (DMMA), fp64 FMA,
cp.async (LDGSTS), shuffles.
python scripts/sass_opcodes.py [lib.so] > profiles/r02_sass_opcodes.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2604_25378_b200/_build/libmvsk_b200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
KEYS = ["UBLKCP", "UTMALDG", "UTMASTG", "SYNCS", "DMMA", "DFMA", "DADD", "DMUL", "LDGSTS", "SHFL", "UCGABAR",
        "MEMBAR", "ATOMS", "REDUX", "LDS", "STS", "LDG", "STG", "BAR"]
kern = None
counts = collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    if kern is None:
        continue
    m = re.search(r"/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if m:
        op = m.group(1).split(".")[0]
        for k in KEYS:
            if op == k or (k == "SYNCS" and op.startswith("SYNCS")) or (k == "BAR" and op == "BAR"):
                counts[kern][k] += 1


def short(name):
    s = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    s = s.replace("mvsk_b200::", "").replace("(anonymous namespace)::", "")
    return s[:110]


print("kernel | " + " ".join(KEYS))
for k, c in counts.items():
    if sum(c.values()) == 0:
        continue
    print(short(k))
    print("    " + "  ".join(f"{key}={c[key]}" for key in KEYS if c[key]))
