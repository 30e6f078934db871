"""Independent-route reference values shared by the oracle pins (no oracle code)."""
import numpy as np
from scipy import integrate

FOUR_PI = 4 * np.pi
MU0 = 4e-7 * np.pi


def box_integral(a, b, c):
    """(1/4pi) int int_{box^2} 1/|r-r'| for an a x b x c box of unit voxels.

    = (8/4pi) int_0^a int_0^b int_0^c (a-x)(b-y)(c-z)/r; the z integral is done
    analytically, int_0^c (c-z)/sqrt(rho^2+z^2) dz = c asinh(c/rho) - sqrt(rho^2+c^2) + rho,
    and the (x,y) integral by adaptive QUADPACK (scipy dblquad).
    """
    def f(y, x):
        rho = np.hypot(x, y)
        inner = c * np.arcsinh(c / rho) - np.sqrt(rho ** 2 + c ** 2) + rho
        return (a - x) * (b - y) * inner
    val, err = integrate.dblquad(f, 0, a, 0, b, epsabs=1e-14, epsrel=1e-13)
    return 8 * val / FOUR_PI


def two_fluid_ab(sigma0, lam, w):
    """Eq. 22-23 retyped for the closed forms (lambda = inf -> normal conductor)."""
    if np.isinf(lam):
        return 1.0 / sigma0, 0.0
    g = w * MU0 * lam ** 2
    den = 1 + (sigma0 * g) ** 2
    return sigma0 * g ** 2 / den, lam ** 2 / den


def bar_closed_form(n, ny, nz, dx, sigma0, lam, f):
    """Uniform-current bar (P8/P9 of SURVEY 8(c)): L = mu0 b l/A + mu0 dx S_box/(ny nz)^2,
    R = a l / A; exact when the uniform J_x is the solution (1x1 and 2x2 cross sections)."""
    w = 2 * np.pi * f
    a, b = two_fluid_ab(sigma0, lam, w)
    l_over_A = n / (ny * nz * dx)
    S = box_integral(n, ny, nz)
    return MU0 * b * l_over_A + MU0 * dx * S / (ny * nz) ** 2, a * l_over_A
