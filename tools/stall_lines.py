"""Aggregate ncu per-SASS stall samples (ncu --page source --print-source sass --csv)
by CUDA source line, using nvdisasm -g line info of the same cubin.
usage: stall_lines.py <sass.csv> <nvdisasm -g output> <kernel mangled name> [top]"""
import csv
import re
import sys
from collections import defaultdict


def line_map(dis, kern):
    txt = open(dis).read()
    i = txt.find(".text." + kern)
    j = txt.find(".section", i + 100)
    cur, out = None, {}
    for l in txt[i:j].splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            # with nvdisasm -gi: the outermost call site in the kernel's own files
            sites = re.findall(r'"([^"]+)", line (\d+)', l)
            own = [x for x in sites if "floe_v3" in x[0] or "floe_v2" in x[0]]
            pick = own[-1] if own else sites[0]
            cur = f"{pick[0].split('/')[-1]}:{pick[1]}"
        m = re.match(r"\s*/\*([0-9a-f]+)\*/", l)
        if m and cur:
            out[int(m.group(1), 16)] = cur
    return out


def main():
    csvf, dis, kern = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    lm = line_map(dis, kern)
    rows = list(csv.reader(open(csvf)))
    hdr = rows[1]
    idx = {h: k for k, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = defaultdict(lambda: defaultdict(float))
    total = 0.0
    base = None
    for r in rows[2:]:
        try:
            addr = int(r[idx["Address"]], 16)
        except (ValueError, KeyError):
            continue
        if base is None:
            base = addr
        addr -= base
        ln = lm.get(addr, "?")
        s = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        agg[ln]["_all"] += s
        total += s
        for c in stall_cols:
            v = r[idx[c]]
            if v:
                agg[ln][c] += float(v)
    items = sorted(agg.items(), key=lambda kv: -kv[1]["_all"])[:top]
    print(f"total samples {total:.0f}")
    for ln, d in items:
        tops = sorted(((v, c) for c, v in d.items() if c != "_all"), reverse=True)[:3]
        print(f"{ln:24s} {d['_all']:8.0f} ({100 * d['_all'] / total:4.1f}%)  " +
              "  ".join(f"{c[6:]}={v:.0f}" for v, c in tops))


if __name__ == "__main__":
    main()
