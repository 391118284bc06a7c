"""Count the Blackwell-specific SASS opcodes per kernel of libmp.so.

    python tools/sass_summary.py [out.json]

Runs `cuobjdump -sass` on the built library and counts, per function, the
opcodes that prove the sm_100a path: UTCHMMA (tcgen05.mma), UTMALDG /
UTMASTG / UTMAREDG (TMA load / store / reduce-add), LDTM / STTM (TMEM
load / store), LDGMC (multimem.ld_reduce over NVSwitch), MUFU.EX2 / TANH,
and HMMA (legacy mma.sync; none expected).
"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2104_04473_b200", "lib", "libmp.so")
KEYS = ["UTCHMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UTMAREDG", "LDTM", "STTM", "HMMA", "MUFU.EX2", "MUFU.TANH",
        "REDG", "LDGMC", "STGMC", "REDGMC"]


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "sass_summary.json")
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    cur, counts = None, collections.defaultdict(collections.Counter)
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if cur and m:
            for k in KEYS:
                if m.group(1).startswith(k):
                    counts[cur][k] += 1
                    break
    tot, rows = collections.Counter(), []
    for fn, c in counts.items():
        tot.update(c)
        if any(c[k] for k in ("UTCHMMA", "UTMALDG", "LDTM", "LDGMC")):
            name = subprocess.run(["c++filt", fn], capture_output=True, text=True).stdout.strip()
            rows.append({"function": name[:120], "counts": dict(c)})
    out = {"library": os.path.relpath(LIB, ROOT), "how": "cuobjdump -sass; opcode-prefix counts per function",
           "totals": dict(tot), "functions": sorted(rows, key=lambda r: r["function"])}
    json.dump(out, open(out_path, "w"), indent=1)
    print(json.dumps(out["totals"]))


if __name__ == "__main__":
    main()
