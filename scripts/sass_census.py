"""SASS instruction census of the tcgen05 kernels (from `cuobjdump -sass`
of libls_b200.so): per kernel, the count of the mnemonics that prove the
tcgen05 / TMEM / TMA path (UTCHMMA, UTCBAR, LDTM, UTMALDG, UTMASTG, UTMAREDG,
UBLKCP, SYNCS) next to the instruction total, one line per template
instantiation:
  cuobjdump -sass paper_2205_13603_b200/_lib/libls_b200.so | c++filt > /tmp/sass.txt
  python scripts/sass_census.py /tmp/sass.txt"""
import collections
import re
import sys

KEYS = ("UTCHMMA", "UTCBAR", "UTCATOMSWS", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UTMAREDG", "UTMAPF",
        "UBLKCP", "UBLKRED", "SYNCS", "FFMA", "HMMA", "RED", "ATOM", "BAR", "WARPSYNC")


def main(path):
    kernels = collections.OrderedDict()
    cur = None
    for line in open(path, errors="replace"):
        m = re.match(r"\s*Function : (.+?)\s*$", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[\w.]+)?", line)
        if m:
            kernels[cur][m.group(2)] += 1
            kernels[cur]["_total"] += 1
    for name, c in kernels.items():
        if not any(k in name for k in ("tc_gemm", "tc_conv")):
            continue
        m2 = re.search(r"(tc_gemm_kernel|tc_conv_kernel)(<[^>]*>)?", name)
        short = m2.group(0) if m2 else name
        print(f"{short}: {c['_total']} instructions")
        print("   " + ", ".join(f"{k} {c[k]}" for k in KEYS if c[k]))


if __name__ == "__main__":
    main(sys.argv[1])
