"""Check that no global load precedes griddepcontrol.wait (SASS ACQBULK) in
kernels that call it: a load hoisted above the wait may read a buffer its
predecessor grid is still writing (programmatic dependent launch)."""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2303_02352_b200/libpairamg_b200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
bad = 0
for fn in re.split(r"\n\s*Function : ", out)[1:]:
    name = fn.split("\n", 1)[0].strip()
    body = fn.split("\n")
    if not any("ACQBULK" in l for l in body):
        continue
    for l in body:
        if "ACQBULK" in l:
            break
        if re.search(r"\bLD(G|S)?\.", l) and "LDC" not in l:
            print("load before wait:", name[:90], "|", l.strip()[:80])
            bad += 1
            break
print("kernels with griddepcontrol.wait checked; violations:", bad)
sys.exit(1 if bad else 0)
