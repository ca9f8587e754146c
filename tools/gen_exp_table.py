"""Writes paper_2206_01885_b200/csrc/exp_table2048.inc: 2^(j/2048), j = 0..2047, each correctly
rounded to fp64 (Python decimal at 80 digits, then float(Decimal), which rounds correctly)."""
import os
from decimal import Decimal, getcontext

getcontext().prec = 80
N = 2048
vals = [float(Decimal(2) ** (Decimal(j) / Decimal(N))) for j in range(N)]
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2206_01885_b200", "csrc",
                   "exp_table2048.inc")
with open(out, "w") as f:
    f.write(f"// 2^(j/{N}), j = 0..{N - 1}, each correctly rounded to fp64 (tools/gen_exp_table.py: Python\n")
    f.write("// decimal at 80 digits, then float(Decimal)); the table of exp_neg_fill (h2_internal.cuh)\n")
    f.write(f"static __device__ const double kExp2Tab{N}[{N}] = {{\n")
    for i in range(0, N, 4):
        f.write("    " + ", ".join(v.hex().replace("0x1.", "0x1.").ljust(23) .strip() for v in vals[i:i + 4]) + ",\n")
    f.write("};\n")
