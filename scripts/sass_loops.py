"""Opcode histogram of every innermost loop (backward branch) of a kernel in
the built library, e.g.

    python scripts/sass_loops.py 'k_p2p_pipeILi10ELi256' [--lib path] [--all]

Only loops containing a marker opcode (default MUFU.RSQ64H, i.e. the pair
loops of k_p2p) are shown unless --all is given.  Used to check FP64
instruction counts and spills (LDL/STL) in hot loops before spending GPU time.
"""
import argparse
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def kernel_sass(lib, pattern):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    funcs, cur, name = {}, [], None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if name:
                funcs[name] = cur
            name, cur = m.group(1), []
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m and name:
            cur.append((int(m.group(1), 16), m.group(2).strip()))
    if name:
        funcs[name] = cur
    hits = {k: v for k, v in funcs.items() if re.search(pattern, k)}
    return hits


def opcode(ins):
    toks = ins.split()
    if toks and toks[0].startswith("@"):
        toks = toks[1:]
    return toks[0].split(".")[0] if toks else "?"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("pattern")
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_2212_08284_b200", "libankh_b200.so"))
    ap.add_argument("--marker", default="MUFU.RSQ64H")
    ap.add_argument("--all", action="store_true")
    a = ap.parse_args()
    for name, ins in kernel_sass(a.lib, a.pattern).items():
        print(name)
        addr_idx = {ad: i for i, (ad, _) in enumerate(ins)}
        loops = []
        for i, (ad, txt) in enumerate(ins):
            m = re.search(r"BRA(?:\.\S+)?\s+(?:!?U?P\d,\s*)?0x([0-9a-f]+)", txt)
            if m:
                tgt = int(m.group(1), 16)
                if tgt <= ad and tgt in addr_idx:
                    loops.append((addr_idx[tgt], i))
        # innermost: no other loop strictly inside
        inner = [l for l in loops if not any(o != l and o[0] >= l[0] and o[1] <= l[1] for o in loops)]
        for lo, hi in inner:
            body = [t for _, t in ins[lo:hi + 1]]
            if not a.all and not any(a.marker in t for t in body):
                continue
            c = collections.Counter(opcode(t) for t in body)
            fp64 = sum(c[k] for k in ("DFMA", "DMUL", "DADD"))
            print(f"  loop 0x{ins[lo][0]:x}-0x{ins[hi][0]:x}: {len(body)} instr, FP64 {fp64} "
                  f"(DFMA {c['DFMA']} DMUL {c['DMUL']} DADD {c['DADD']}), LDL {c['LDL']} STL {c['STL']}")
            print("    " + " ".join(f"{k}:{v}" for k, v in c.most_common()))


if __name__ == "__main__":
    main()
