#!/bin/bash
# Compile gemm.cu (worktree) with extra flags and print the promotion loop's instruction order for one
# kernel instantiation, condensed: runs of FFMA2/FMUL2 are collapsed to a count, and TMEM loads,
# barrier waits/arrives, shared loads and branches are shown in place.  Experiments only.
#   tools/sass_order.sh <kernel-regex, e.g. 'k_gemm_bsILb0ELb0ELb0ELb1E'> [nvcc flags...]
set -e
K=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -prec-div=true -ftz=false --expt-relaxed-constexpr \
     -I $ROOT/include "$@" -cubin -o $TMP/g.cubin $ROOT/paper_2412_19437_b200/csrc/gemm.cu
cuobjdump -sass $TMP/g.cubin | awk -v k="$K" '$0 ~ "Function : .*"k {p=1; next} p && /Function : / {p=0} p' \
  | sed 's@/\* 0x[0-9a-f]* \*/@@' > $TMP/k.sass
# promotion loop = the block containing the first LDTM, from the preceding backward-branch target
python3 - "$TMP/k.sass" <<'EOF'
import re, sys
lines = [l.strip() for l in open(sys.argv[1]) if re.match(r"\s*/\*[0-9a-f]{4}\*/", l)]
ins = []
for l in lines:
    m = re.match(r"/\*([0-9a-f]+)\*/\s+(.*?)\s*;", l)
    if m: ins.append((int(m.group(1), 16), m.group(2)))
first = next(i for i, (a, t) in enumerate(ins) if "LDTM" in t)
# loop back-edge: first "BRA.U UP0, <target>" after the LDTM with target < LDTM address
back = next(i for i in range(first, len(ins)) if re.match(r"(@\S+ )?BRA(\.U)? .*0x([0-9a-f]+)$", ins[i][1])
            and int(re.search(r"0x([0-9a-f]+)$", ins[i][1]).group(1), 16) < ins[first][0])
tgt = int(re.search(r"0x([0-9a-f]+)$", ins[back][1]).group(1), 16)
start = next(i for i, (a, t) in enumerate(ins) if a == tgt)
body = ins[start:back + 1]
print(f"loop {hex(tgt)}..{hex(ins[back][0])}: {len(body)} instructions")
from collections import Counter
c = Counter(t.split()[0].lstrip("@!P0123456789 ").split(".")[0] if not t.startswith("@") else t.split()[1].split(".")[0] for _, t in body)
print("  " + ", ".join(f"{k} {v}" for k, v in c.most_common()))
run = 0
out = []
for a, t in body:
    op = t.split()[1] if t.startswith("@") else t.split()[0]
    if op.startswith(("FFMA2", "FMUL2", "FFMA", "FMUL")):
        run += 1; continue
    if any(s in t for s in ("LDTM", "SYNCS", "LDS", "BRA", "ELECT", "BAR", "STS", "UTMA", "UBLKCP")):
        if run: out.append(f"[{run} fma]"); run = 0
        out.append(t[:70])
if run: out.append(f"[{run} fma]")
print("\n".join("  " + o for o in out))
EOF
rm -rf $TMP
