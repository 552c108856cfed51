"""Probe the 128B-swizzled MN-major tf32 convention."""
import subprocess, sys
sys.path.insert(0, ".")
CODE = open("tools/tf32_probe.py").read().split("CODE = r'''")[1].split("'''")[0]
# p = [kr, sk, sk_in, mr, sm, sm_in, lbo, sbo, kstep, mn, swz, layout_type]
atom = 8 * 128  # 1 KB atom: 8 k-rows x 128 B (32 mn)
cands = []
for sm, sk in ((atom, 4 * atom), (4 * atom, atom)):   # mn-atoms adjacent / k-atoms adjacent (M=128: 4 mn atoms, K=32: 4 k atoms)
    for lbo, sbo in ((sm, sk), (sk, sm), (sm, 1024), (1024, sm), (sk, 1024), (16, sm), (sm, 16), (16, sk), (sk, 16)):
        for lt in (2, 1):
            cands.append([8, sk, 0, 32, sm, 0, lbo, sbo, sk, 1, 1, lt])
for p in cands:
    r = subprocess.run([sys.executable, "-c", CODE, str(p)], capture_output=True, text=True, timeout=60)
    out = [l for l in r.stdout.splitlines() if l.startswith("ERR")]
    err = float(out[0].split()[1]) if out else None
    print(p, err, flush=True)
