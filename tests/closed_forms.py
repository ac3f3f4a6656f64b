"""Closed forms that pin the oracle's G(tau) quadrature (test-side only).

G(tau) = int_0^tau dt' int_0^t' dt'' alpha(t'-t'')  with alpha from Eq. 4
       = (1/pi) int_0^inf dw J(w)/w^2 [coth(w/2kT)(1 - cos w tau) - i (w tau - sin w tau)].

Each closed form below is derived independently of the quadrature (series /
special-function identities evaluated with mpmath at 30 digits):

* Ohmic-exp J = (pi/2) xi w e^{-w/wc}:
    T = 0 (Frullani):  G0 = (xi/2) [ln(1 + i wc tau) - i wc tau]
    T > 0: coth(x/2) = 1 + 2 sum_n e^{-n x} and int_0^inf e^{-aw}(1-cos w tau)/w dw = (1/2) ln(1+tau^2/a^2) give
           G = G0 + (xi/2) sum_{n>=1} ln(1 + tau^2/(1/wc + n beta)^2)
             = G0 + xi [ln Gamma(1+c) - Re ln Gamma(1+c+ix)],  c = 1/(beta wc), x = tau/beta
    (Euler product  prod_{n>=1} (1 + x^2/(n+c)^2) = |Gamma(1+c)|^2 / |Gamma(1+c+ix)|^2).
* Debye J = (pi/2) xi w wc^2/(w^2+wc^2): Matsubara expansion of coth gives, for t > 0,
    alpha(t) = (pi xi c^2/4)[cot(beta c/2) - i] e^{-ct} + (pi xi c^2/beta) sum_n nu_n e^{-nu_n t}/(nu_n^2 - c^2),
    nu_n = 2 pi n / beta,  and  int_0^tau (tau-u) e^{-g u} du = tau/g - (1-e^{-g tau})/g^2.
    The n >= n0 tail is summed with Hurwitz zeta functions.
* super-Ohmic Gaussian J = A w^3 e^{-(w/wc)^2} (Eq. 21, reading C.3-5), T = 0:
    int_0^inf w e^{-w^2/c^2} dw = c^2/2,  int w^2 e^{-w^2/c^2} = sqrt(pi) c^3/4,
    int w e^{-w^2/c^2} cos(w tau) = (c^2/2)(1 - c tau D(c tau/2)) (D = Dawson),
    int w e^{-w^2/c^2} sin(w tau) = (sqrt(pi)/4) c^3 tau e^{-c^2 tau^2/4}.
  T > 0: 30-digit mpmath quadrature of the (smooth, Gaussian-damped) integrand.
"""
from __future__ import annotations

import mpmath as mp

mp.mp.dps = 30


def G_ohmic(xi, wc, kT, tau) -> complex:
    xi, c, tau = mp.mpf(xi), mp.mpf(wc), mp.mpf(tau)
    g0 = xi / 2 * (mp.log(1 + 1j * c * tau) - 1j * c * tau)
    if kT == 0:
        return complex(g0)
    beta = 1 / mp.mpf(kT)
    cc, x = 1 / (beta * c), tau / beta
    return complex(g0 + xi * (mp.loggamma(1 + cc) - mp.re(mp.loggamma(1 + cc + 1j * x))))


def G_debye(xi, wc, kT, tau, n0: int = 1000) -> complex:
    beta, xi, c, tau = 1 / mp.mpf(kT), mp.mpf(xi), mp.mpf(wc), mp.mpf(tau)
    a = 2 * mp.pi / beta

    def phi(g):
        return tau / g - (1 - mp.exp(-g * tau)) / g**2

    pre = mp.pi * xi * c**2 / 4 * (mp.cot(beta * c / 2) - 1j) * phi(c)
    s = mp.fsum((a * n) / ((a * n) ** 2 - c**2) * phi(a * n) for n in range(1, n0))
    # n >= n0: nu/(nu^2-c^2) (tau/nu - 1/nu^2) = sum_m c^{2m}(tau/nu^{2m+2} - 1/nu^{2m+3}); e^{-nu tau} negligible
    s += mp.fsum(c ** (2 * m) * (tau * mp.zeta(2 * m + 2, n0) / a ** (2 * m + 2) - mp.zeta(2 * m + 3, n0) / a ** (2 * m + 3))
                 for m in range(16))
    return complex(pre + mp.pi * xi * c**2 / beta * s)


def G_superohmic(A, wc, kT, tau) -> complex:
    A, c, tau = mp.mpf(A), mp.mpf(wc), mp.mpf(tau)
    if kT == 0:
        re = c**2 / 2 - c**2 / 2 * (1 - c * tau * (mp.sqrt(mp.pi) / 2 * mp.exp(-(c * tau / 2) ** 2) * mp.erfi(c * tau / 2)))
        im_wt = tau * mp.sqrt(mp.pi) * c**3 / 4
        im_sin = mp.sqrt(mp.pi) / 4 * c**3 * tau * mp.exp(-(c**2) * tau**2 / 4)
        return complex(A / mp.pi * (re - 1j * (im_wt - im_sin)))
    kT = mp.mpf(kT)

    def fr(w):
        return A * w * mp.exp(-((w / c) ** 2)) * mp.coth(w / (2 * kT)) * 2 * mp.sin(w * tau / 2) ** 2 / mp.pi

    def fi(w):
        return -A * w * mp.exp(-((w / c) ** 2)) * (w * tau - mp.sin(w * tau)) / mp.pi

    pts = [mp.mpf(0)] + [c * k / 2 for k in range(1, 41)]
    return complex(mp.quad(fr, pts) + 1j * mp.quad(fi, pts))
