"""SASS mnemonic counts per kernel of the built library (runs without a GPU):

    python tools/sass_evidence.py > profiles/r2/sass_evidence.txt

UBLKCP = TMA bulk copy (cp.async.bulk), UBLKPF = bulk L2 prefetch, SYNCS =
mbarrier ops, FADD2/FMUL2/FFMA2 = paired fp32, F2FP.BF16 = RNE bf16 pack,
PRMT = byte permute, STG.E*.128 = 16 B stores (EF = evict-first), LDS/STS =
shared memory, ATOMG/RED = global atomics, MEMBAR = fences."""
import re
import subprocess
import sys
from collections import Counter, OrderedDict

LIB = "paper_2409_18749_b200/libtsb200.so"
KEEP = ("UBLKCP", "UBLKPF", "SYNCS", "FADD2", "FMUL2", "FFMA2", "F2FP.BF16", "PRMT",
        "STG.E.128", "STG.E.EF.128", "STG.E.STRONG.SYS", "LDG.E.128", "LDS", "LDS.128", "STS",
        "ATOMG", "RED", "MEMBAR", "SHFL", "LOP3")
PREFIX = ("UBLKCP", "UBLKPF", "SYNCS", "LDS", "STS", "MEMBAR", "ATOMG", "RED", "SHFL", "LOP3")


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    kernels: "OrderedDict[str, Counter]" = OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m and cur:
            op = m.group(1)
            if op in KEEP:
                kernels[cur][op] += 1
            elif op.split(".")[0] in PREFIX:
                kernels[cur][op.split(".")[0]] += 1
    print(__doc__.strip().splitlines()[0])
    print(f"source: cuobjdump -sass {LIB} (sm_100a)\n")
    for name, c in kernels.items():
        short = re.sub(r"^_ZN\d+_GLOBAL__N__[0-9a-f_]+\d+", "", name)[:90]
        print(f"{short}: " + ", ".join(f"{k}={c[k]}" for k in KEEP if c[k]))


if __name__ == "__main__":
    sys.exit(main())
