"""Fit of the forward GELU used by the pass C epilogues (csrc/kernels.cuh gelu_f):
    Phi(z) = 1 / (1 + 2^(z * P(min(z^2, 5.5^2)))),  P a degree-6 polynomial,
i.e. a logistic form whose logit/z is fitted in u = z^2 by iteratively
reweighted least squares toward the minimax error in z*Phi(z).  Prints the
coefficients and the fp32 error against z * scipy.special.ndtr(z) (fp64)."""
import numpy as np
from scipy.special import ndtr

R, n = 5.5, 7
z = np.cos(np.linspace(0, np.pi, 20000)) * R / 2 + R / 2
z = z[z > 1e-4]
Phi = ndtr(z)
lg = np.log(Phi / (1 - Phi)) / z
V = np.vander(z * z, n, increasing=True)
w = Phi * (1 - Phi) * z
coef, *_ = np.linalg.lstsq(V * w[:, None], lg * w, rcond=None)
for _ in range(30):
    err = np.abs(1 / (1 + np.exp(-z * (V @ coef))) - Phi) * z
    w2 = w * (1 + (err / err.max()) ** 2 * 50)
    coef, *_ = np.linalg.lstsq(V * w2[:, None], lg * w2, rcond=None)
c32 = (-coef * np.log2(np.e)).astype(np.float32)
print("coefficients (exp2 form, u^0..u^6):", [repr(float(x)) for x in c32])
zz = np.linspace(-10, 10, 2000001).astype(np.float32)
uu = np.minimum(zz * zz, np.float32(R * R))
acc = np.full_like(uu, c32[-1])
for k in range(n - 2, -1, -1):
    acc = (acc * uu + c32[k]).astype(np.float32)
g = (zz * (np.float32(1) / (np.float32(1) + np.exp2(zz * acc)))).astype(np.float32)
ref = zz.astype(np.float64) * ndtr(zz.astype(np.float64))
m = np.abs(ref) > 0.05
print("max |GELU error| %.2e, max relative error where |GELU| > 0.05: %.2e"
      % (np.max(np.abs(g - ref)), np.max(np.abs(g - ref)[m] / np.abs(ref[m]))))
