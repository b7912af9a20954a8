"""Constants of ozaki_engine.cuh exp_tab256: 2^(j/256), j = 0..255, correctly rounded to fp64 (60-digit
Decimal, each value checked against its two neighbours), and the scaled Taylor coefficients
L^k / k! of e^{r' L} - 1 with L = ln2/256.  Prints C source."""
import math
from decimal import Decimal, getcontext

getcontext().prec = 60
ln2 = Decimal(2).ln()
L = ln2 / 256
vals = []
for j in range(256):
    ex = Decimal(2) ** (Decimal(j) / 256)
    v = float(ex)
    for nb in (math.nextafter(v, math.inf), math.nextafter(v, -math.inf)):
        assert abs(Decimal(v) - ex) <= abs(Decimal(nb) - ex)
    vals.append(v)
print("__constant__ double kExp2Tab256[256] = {")
for i in range(0, 256, 4):
    print("    " + ", ".join(repr(v) for v in vals[i:i + 4]) + ",")
print("};")
print(f"kInvL256 = {float(256 / ln2)!r}  // 256 / ln 2")
for k in range(1, 5):
    print(f"C{k} = {float(L ** k / math.factorial(k))!r}  // L^{k}/{k}!")
