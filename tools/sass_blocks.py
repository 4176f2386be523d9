"""Per-basic-block instruction mix of a kernel's SASS (cuobjdump -sass): the blocks that hold MUFU.EX2 (the pair
math of the tensor-core E step), with FP32 lane-ops per pair (f32x2 instructions count 2).  Blocks are split at
branch targets and after branches.  Diagnostic.
python tools/sass_blocks.py <object or .so> [kernel substring] [min MUFU per block]"""
import re
import subprocess
import sys
from collections import Counter

obj = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else "estep_tc_kernelILb0E"
min_mufu = int(sys.argv[3]) if len(sys.argv) > 3 else 16
txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
for part in re.split(r"\n\s*Function : ", txt)[1:]:
    name = part.split("\n", 1)[0]
    if want not in name:
        continue
    ins = [(int(a, 16), b.strip()) for a, b in re.findall(r"/\*([0-9a-f]{4,6})\*/\s+([^;]*);", part)]
    targets = {int(m.group(1), 16) for _, i in ins for m in [re.search(r"\bBRA(?:\.\w+)*\s+(?:!?U?P\w+,\s*)?(0x[0-9a-f]+)", i)] if m}
    blocks, cur, start = [], Counter(), ins[0][0] if ins else 0
    for addr, i in ins:
        if addr in targets and cur:
            blocks.append((start, cur))
            cur, start = Counter(), addr
        op = re.sub(r"^@!?U?P\w+\s+", "", i).split()[0]
        cur["ALL"] += 1
        cur[op.split(".")[0]] += 1
        if op.startswith("MUFU.EX2"):
            cur["EX2"] += 1
        if re.match(r"BRA", op):
            blocks.append((start, cur))
            cur, start = Counter(), addr + 16
    blocks.append((start, cur))
    print(name[:70])
    for start, b in blocks:
        if b["EX2"] >= min_mufu:
            f = b["FFMA2"] + b["FADD2"] + b["FMUL2"]
            ops = 2 * f + b["FFMA"] + b["FADD"] + b["FMUL"]
            print(f"  @{start:#07x}: EX2 {b['EX2']:3d}  FFMA2 {b['FFMA2']:3d} FADD2 {b['FADD2']:3d} FMUL2 {b['FMUL2']:3d} "
                  f"FFMA {b['FFMA']:2d} -> lane-ops/pair {ops / b['EX2']:5.2f} | LOP3 {b['LOP3']:3d} LDS {b['LDS']:3d} "
                  f"STTM {b['STTM']:2d} MOV {b['MOV']:3d} all {b['ALL']:4d} ({b['ALL'] / b['EX2']:.2f}/pair)")
