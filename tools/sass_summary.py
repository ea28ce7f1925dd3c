#!/usr/bin/env python
"""SASS instruction counts of the K6 instantiations in libxct_b200.so (the
evidence that FHFMA / FFMA2 / LDGSTS / LDS.128 / UBLKCP are what runs), plus
registers and spills from the ptxas log.

  python tools/sass_summary.py > profiles/r02_sass_k6.txt
"""
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2009_07226_b200" / "libxct_b200.so"
OPS = ["FHFMA", "FFMA2", "FFMA", "FMUL", "FADD", "HFMA2", "HMUL2", "HADD2", "DFMA", "DMUL",
       "DADD", "LDS.128", "LDS.64", "LDS", "LDGSTS.E.BYPASS.128", "LDGSTS", "LDG.E.NA.128",
       "LDG", "UBLKCP", "SYNCS", "BAR.SYNC", "SHFL"]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True,
                          check=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)[1:]
    log = (ROOT / "build" / "obj" / "spmm.ptxas.log")
    regs = {}
    if log.exists():
        cur = None
        for line in log.read_text().splitlines():
            m = re.search(r"Compiling entry function '(\S+)'", line)
            if m:
                cur = m.group(1)
            m = re.search(r"Used (\d+) registers", line)
            if m and cur:
                regs.setdefault(cur, {})["regs"] = int(m.group(1))
            m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
            if m and cur:
                regs.setdefault(cur, {})["spill"] = f"{m.group(1)}/{m.group(2)} B"
    print(f"# SASS of {LIB.name} (sm_100a), K6 kernels; counts are static instructions")
    for f in funcs:
        name = f.split("\n", 1)[0].strip()
        if "spmm" not in name:
            continue
        body = f.split("\n", 1)[1]
        ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", body)
        c = Counter()
        for i in ins:
            for op in OPS:
                if i == op or i.startswith(op + "."):
                    c[op] += 1
                    break
        short = re.sub(r"_ZN\w+?spmm_cu\w+?(spmm_\w+?kernel)", r"\1", name)
        r = regs.get(name, {})
        print(f"\n{short}\n  total {len(ins)} instructions, registers {r.get('regs', '?')}, "
              f"spill {r.get('spill', '?')}")
        print("  " + ", ".join(f"{k} {v}" for k, v in c.most_common() if v))


if __name__ == "__main__":
    sys.exit(main())
