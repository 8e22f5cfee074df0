"""Count DMMA / NOP / LDS in the unpredicated main loop of a kernel's SASS (offline check of
the DMMA issue pattern).  usage: python tools/sass_loop.py lib.so mangled_name"""
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-sass", "-fun", sys.argv[2], sys.argv[1]], capture_output=True, text=True).stdout
ins = [l.split(";")[0].strip() for l in out.splitlines() if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l)]
ins = [re.sub(r"^/\*[0-9a-f]+\*/\s*", "", l) for l in ins]
dm = [i for i, l in enumerate(ins) if "DMMA" in l]
print("total instr", len(ins), "DMMA", len(dm), "NOP", sum("NOP" in l for l in ins))
# longest run between first and last DMMA of the densest window
gaps = [dm[i + 1] - dm[i] - 1 for i in range(len(dm) - 1)]
seg = ins[dm[0]:dm[-1] + 1] if dm else []
print("in DMMA span: NOP", sum("NOP" in l for l in seg), "LDS", sum("LDS" in l for l in seg), "other",
      sum(not any(k in l for k in ("NOP", "LDS", "DMMA")) for l in seg))
if len(sys.argv) > 3:
    for l in seg[: int(sys.argv[3])]:
        print("   ", l)
