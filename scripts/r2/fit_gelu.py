"""Fit of the GEMM GELU epilogue's erfc (block.cu gelu2): for u = |x|/sqrt(2)
clamped to [0, 4.5], erfc(u) = 2^(Q(u) - u^2 log2 e) with Q(u) = log2(erfc(u)
e^(u^2)) a degree-11 polynomial (Chebyshev fit, power basis, fp32
coefficients).  Prints the coefficients and the max relative error of the
fp32 Horner evaluation against scipy's erfc; the GELU is then
0.5 x (x < 0 ? E : 2 - E), exact GELU to ~4e-6 relative (bf16 ulp: 3.9e-3)."""
import numpy as np
from scipy.special import erfc

U, DEG = 4.5, 11
L2E = np.log2(np.e)
k = np.arange(4000)
u = (U / 2) * (1 - np.cos(np.pi * (k + 0.5) / 4000))
Q = np.log2(erfc(u)) + u * u * L2E
c = np.polynomial.chebyshev.Chebyshev.fit(u, Q, DEG, domain=[0, U]).convert(kind=np.polynomial.Polynomial).coef
c32 = c.astype(np.float32)
uu = np.linspace(0, U, 400001).astype(np.float32)
acc = np.full_like(uu, c32[-1])
for a in c32[-2::-1]:
    acc = (acc * uu + a).astype(np.float32)
arg = (acc - (uu * uu).astype(np.float32) * np.float32(L2E)).astype(np.float32)
rel = np.abs(np.exp2(arg.astype(np.float64)) / erfc(uu.astype(np.float64)) - 1).max()
print("coefficients (c0 .. c11):")
print(", ".join(f"{float(v):.9e}f" for v in c32))
print(f"max relative error of erfc on [0, {U}]: {rel:.2e}")
