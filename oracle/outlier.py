"""Oracle: outlier-weight estimation and confidence filtering (§3.2-3.3).  TEST INFRASTRUCTURE ONLY.

* Eq. 7: with the true alignment the expected outlier count Σ_n P(M+1|g*(x_n)) equals ηN;
  bounding p(g*(x_n)|m) by its maximum c_m (Eq. 2) gives the upper bound
      w_max = η V Σ_m π(m) c_m / ((1 - η) + η V Σ_m π(m) c_m),
  and the paper sets w_0 = w_max.  c_m = √(1+α_m)/(2πσ²)^{3/2} (consistent normaliser, reading
  R1) or 1/(2πσ²)^{3/2} (Eq. 9-10 literal).  c_m depends on σ², so w_0 is re-evaluated at every EM
  iteration from the current σ² (reading R22).
* Eq. 8: φ(x) = e_min / e(x); π(m) = φ(y_m)/Σ_m φ(y_m); w_n = 1 - (1 - w_0) φ(x_n);
  points with φ below a threshold are truncated.
* Depth error model (reading R23): e(z) = c0 + c1 z² of the camera-frame depth z, with the
  RGBD config's noise model sd = 0.002 z² (c0 = 0, c1 = 0.002) and e_min = e(z_min) at the sensor's
  minimum range z_min = 0.4 m; φ is clipped to [0, 1].
"""
from __future__ import annotations

import numpy as np


def component_normalizer(alpha, sigma2: float, consistent: bool = True):
    """c_m of Eq. 2: √(1+α_m)/(2πσ²)^{3/2}; without the √(1+α_m) factor in the literal mode."""
    alpha = np.asarray(alpha, dtype=np.float64)
    base = (2.0 * np.pi * sigma2) ** -1.5
    return base * np.sqrt(1.0 + alpha) if consistent else np.full_like(alpha, base)


def outlier_weight_max(eta: float, V: float, prior, alpha, sigma2: float, consistent: bool = True) -> float:
    """w_max of §3.2: η V Σπc / ((1 - η) + η V Σπc)."""
    if not 0.0 <= eta < 1.0:
        raise ValueError("eta must lie in [0, 1)")
    s = float(np.dot(np.asarray(prior, dtype=np.float64), component_normalizer(alpha, sigma2, consistent)))
    a = eta * V * s
    return a / ((1.0 - eta) + a)


def expected_outliers(post_out) -> float:
    """E(N_outlier) = Σ_n P(M+1 | x_n) (Eq. 7)."""
    return float(np.sum(post_out))


def confidence_prior(phi_y):
    """π(m) = φ(y_m) / Σ_m φ(y_m) (Eq. 8)."""
    phi_y = np.asarray(phi_y, dtype=np.float64)
    s = phi_y.sum()
    if not s > 0.0:
        raise ValueError("all-zero target confidences")
    return phi_y / s


def point_outlier_weights(w0: float, phi_x):
    """w_n = 1 - (1 - w_0) φ(x_n) (Eq. 8)."""
    return 1.0 - (1.0 - w0) * np.asarray(phi_x, dtype=np.float64)


def depth_confidence(z, c0: float = 0.0, c1: float = 0.002, z_min: float = 0.4):
    """φ = e_min / e(z), e(z) = c0 + c1 z², e_min = e(z_min); clipped to [0, 1] (reading R23)."""
    z = np.asarray(z, dtype=np.float64)
    e = c0 + c1 * z * z
    return np.clip((c0 + c1 * z_min * z_min) / e, 0.0, 1.0)


def truncate(points, phi, threshold: float):
    """Keep the points with φ ≥ threshold, in their original order."""
    keep = np.asarray(phi) >= threshold
    return np.asarray(points)[keep], np.asarray(phi)[keep], keep
