"""Per-kernel SASS instruction counts of the product library (the opcodes that
prove which hardware paths a kernel uses: tcgen05 MMAs, TMEM loads, bulk
copies, legacy tensor-core MMAs, mbarrier ops), from cuobjdump -sass.

    python tools/sass_summary.py [paper_2505_05950_b200/libfloe_b200.so] > profiles/rNN_sass_summary.json
"""
import json
import re
import subprocess
import sys
from collections import Counter

OPS = ["UTCIMMA", "UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "UBLKPF", "UTMALDG",
       "IMMA", "HMMA", "SYNCS", "REDG", "ATOMG", "BAR", "MEMBAR", "FFMA2", "FFMA", "LDS", "LDG", "LDL",
       "STL"]


def main():
    so = sys.argv[1] if len(sys.argv) > 1 else "paper_2505_05950_b200/libfloe_b200.so"
    txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, check=True).stdout
    kernels = {}
    cur = None
    for line in txt.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            op = m.group(1)
            kernels[cur]["_instructions"] += 1
            if op in OPS:
                kernels[cur][op] += 1
    demangled = {}
    names = list(kernels)
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    for raw, nice in zip(names, out.splitlines()):
        demangled[nice.split("(")[0]] = dict(sorted(kernels[raw].items()))
    keep = {k: v for k, v in demangled.items()
            if k.startswith(("floe_v3", "floe_v2", "floe_tc", "floe_bl", "floe_cal", "floe_k", "floe_gen"))
            or "floe" in k}
    json.dump({"source": so, "tool": "cuobjdump -sass (sm_100a)", "kernels": keep}, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
