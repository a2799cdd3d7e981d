"""Per-kernel SASS instruction counts that prove the Blackwell paths
(tcgen05 MMA = UTCHMMA / UTCQMMA, TMEM ld/st = LDTM / STTM, TMA = UTMALDG /
UTMASTG / UBLKCP, packed FP32 = FFMA2 / FADD2 / FMUL2, PDL = griddepcontrol)
from the built objects: python tools/sass_summary.py build/obj/*.o"""
import collections
import re
import subprocess
import sys

KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "SYNCS", "FFMA2", "FADD2",
        "FMUL2", "ACQBULK", "LDS", "STS", "LDG", "STG", "SHFL", "MUFU", "DFMA"]


def main(paths):
    for path in paths:
        sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
        kern, counts = None, collections.Counter()
        out = []
        for line in sass.splitlines():
            m = re.match(r"\s+Function : (\S+)", line)
            if m:
                if kern:
                    out.append((kern, counts))
                kern, counts = m.group(1), collections.Counter()
                continue
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
            if m and kern:
                op = m.group(1)
                for k in KEYS:
                    if op == k or op.startswith(k + "."):
                        counts[k] += 1
                counts["total"] += 1
        if kern:
            out.append((kern, counts))
        for k, c in out:
            short = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()[:110]
            tags = " ".join(f"{key}={c[key]}" for key in KEYS if c[key])
            print(f"{path.split('/')[-1]:<16} {short}\n    total={c['total']} {tags}")


if __name__ == "__main__":
    main(sys.argv[1:])
