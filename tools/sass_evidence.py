"""Per-kernel SASS instruction evidence from libparrot_b200.so: tcgen05 MMAs
(UTC*MMA), TMA loads (UTMALDG), TMEM loads (LDTM), cp.async (LDGSTS).

    python tools/sass_evidence.py > profiles/r1_sass.md
"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2303_01778_b200/libparrot_b200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
kernels = collections.OrderedDict()
cur = None
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        kernels[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    for tag, pat in (("UTC*MMA", r"\bUTC\w*MMA\b"), ("UTMALDG", r"\bUTMALDG\b"), ("LDTM", r"\bLDTM\b"),
                     ("LDGSTS", r"\bLDGSTS\b"), ("UBLKCP/UBLKRED", r"\bUBLK\w+\b")):
        if re.search(pat, line):
            kernels[cur][tag] += 1
demangled = subprocess.run(["c++filt"], input="\n".join(kernels), capture_output=True, text=True).stdout.split("\n")
print("# SASS evidence (`cuobjdump -sass libparrot_b200.so`), static instruction counts\n")
print("| kernel | UTC*MMA | UTMALDG | LDTM | LDGSTS | UBLK* |")
print("|---|---|---|---|---|---|")
for (name, c), dn in zip(kernels.items(), demangled):
    if not any(c.values()):
        continue
    short = re.sub(r"\(.*", "", dn.replace("(anonymous namespace)::", "").replace("void ", ""))
    print(f"| `{short}` | {c['UTC*MMA']} | {c['UTMALDG']} | {c['LDTM']} | {c['LDGSTS']} | {c['UBLK/UBLKRED'] if False else c['UBLKCP/UBLKRED']} |")
