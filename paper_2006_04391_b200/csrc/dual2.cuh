// dual2.cuh -- second-order forward dual with an inner direction (d1) and an
// outer family of six directions (d2) plus the mixed second derivatives
// (d12): gsmkit ad.py:134-239 (Dual2).  Arithmetic restates the reference
// operation by operation (division is multiplication by the reciprocal,
// ad.py:184-198); plain doubles (D<0>) act as the reference's float
// operands.  Used by the Rosenbrock integrator's jac_dir2 (odeint.py:306-337)
// through the semi-automatic hand partials (semi.cuh).  Host + device.
#pragma once

#include "ad.cuh"

namespace am {

// NO outer directions: 6 (one thread per point) or 1 (one lane per
// sensitivity column, adaptive.cuh lane groups)
template <int NO>
struct D2T {
    double v, d1;
    double d2[NO], d12[NO];
};
using D2 = D2T<6>;

template <int NO>
AM_HD D2T<NO> operator+(const D2T<NO>& x, const D2T<NO>& y) {
    D2T<NO> r;
    r.v = x.v + y.v;
    r.d1 = x.d1 + y.d1;
    for (int k = 0; k < NO; ++k) {
        r.d2[k] = x.d2[k] + y.d2[k];
        r.d12[k] = x.d12[k] + y.d12[k];
    }
    return r;
}
template <int NO>
AM_HD D2T<NO> operator+(const D2T<NO>& x, const D<0>& o) {
    D2T<NO> r = x;
    r.v = x.v + o.v;
    return r;
}
template <int NO>
AM_HD D2T<NO> operator+(const D<0>& o, const D2T<NO>& x) { return x + o; }  // __radd__ = __add__
template <int NO>
AM_HD D2T<NO> operator-(const D2T<NO>& x, const D2T<NO>& y) {
    D2T<NO> r;
    r.v = x.v - y.v;
    r.d1 = x.d1 - y.d1;
    for (int k = 0; k < NO; ++k) {
        r.d2[k] = x.d2[k] - y.d2[k];
        r.d12[k] = x.d12[k] - y.d12[k];
    }
    return r;
}
template <int NO>
AM_HD D2T<NO> operator-(const D2T<NO>& x, const D<0>& o) {
    D2T<NO> r = x;
    r.v = x.v - o.v;
    return r;
}
template <int NO>
AM_HD D2T<NO> operator-(const D<0>& o, const D2T<NO>& x) {  // __rsub__
    D2T<NO> r;
    r.v = o.v - x.v;
    r.d1 = -x.d1;
    for (int k = 0; k < NO; ++k) {
        r.d2[k] = -x.d2[k];
        r.d12[k] = -x.d12[k];
    }
    return r;
}
template <int NO>
AM_HD D2T<NO> operator-(const D2T<NO>& x) {
    D2T<NO> r;
    r.v = -x.v;
    r.d1 = -x.d1;
    for (int k = 0; k < NO; ++k) {
        r.d2[k] = -x.d2[k];
        r.d12[k] = -x.d12[k];
    }
    return r;
}
template <int NO>
AM_HD D2T<NO> operator*(const D2T<NO>& x, const D2T<NO>& y) {
    D2T<NO> r;
    r.v = x.v * y.v;
    r.d1 = x.d1 * y.v + x.v * y.d1;
    for (int k = 0; k < NO; ++k) {
        r.d2[k] = x.d2[k] * y.v + x.v * y.d2[k];
        r.d12[k] = x.d12[k] * y.v + x.d1 * y.d2[k] + x.d2[k] * y.d1 + x.v * y.d12[k];
    }
    return r;
}
template <int NO>
AM_HD D2T<NO> operator*(const D2T<NO>& x, const D<0>& o) {
    D2T<NO> r;
    r.v = x.v * o.v;
    r.d1 = x.d1 * o.v;
    for (int k = 0; k < NO; ++k) {
        r.d2[k] = x.d2[k] * o.v;
        r.d12[k] = x.d12[k] * o.v;
    }
    return r;
}
template <int NO>
AM_HD D2T<NO> operator*(const D<0>& o, const D2T<NO>& x) { return x * o; }  // __rmul__ = __mul__

// _reciprocal (ad.py:184-192)
template <int NO>
AM_HD D2T<NO> reciprocal(const D2T<NO>& x) {
    const double inv = 1.0 / x.v, inv2 = inv * inv;
    D2T<NO> r;
    r.v = inv;
    r.d1 = -x.d1 * inv2;
    for (int k = 0; k < NO; ++k) {
        r.d2[k] = -x.d2[k] * inv2;
        r.d12[k] = -x.d12[k] * inv2 + 2.0 * x.d1 * x.d2[k] * inv2 * inv;
    }
    return r;
}
template <int NO>
AM_HD D2T<NO> operator/(const D2T<NO>& x, const D2T<NO>& y) { return x * reciprocal(y); }
template <int NO>
AM_HD D2T<NO> operator/(const D2T<NO>& x, const D<0>& o) {
    D2T<NO> r;
    r.v = x.v / o.v;
    r.d1 = x.d1 / o.v;
    for (int k = 0; k < NO; ++k) {
        r.d2[k] = x.d2[k] / o.v;
        r.d12[k] = x.d12[k] / o.v;
    }
    return r;
}
template <int NO>
AM_HD D2T<NO> operator/(const D<0>& o, const D2T<NO>& x) { return reciprocal(x) * o; }  // __rtruediv__

// Dual2.__pow__ (ad.py:207-215)
template <int NO>
AM_HD D2T<NO> dpow(const D2T<NO>& x, double c) {
    const double f1 = c * ::pow(x.v, c - 1.0);
    const double f2 = c * (c - 1.0) * ::pow(x.v, c - 2.0);
    D2T<NO> r;
    r.v = ::pow(x.v, c);
    r.d1 = f1 * x.d1;
    for (int k = 0; k < NO; ++k) {
        r.d2[k] = f1 * x.d2[k];
        r.d12[k] = f1 * x.d12[k] + f2 * x.d1 * x.d2[k];
    }
    return r;
}
// Dual2.sqrt (ad.py:217-220)
template <int NO>
AM_HD D2T<NO> dsqrt(const D2T<NO>& x) {
    const double s = ::sqrt(x.v), g = 0.5 / s;
    D2T<NO> r;
    r.v = s;
    r.d1 = g * x.d1;
    for (int k = 0; k < NO; ++k) {
        r.d2[k] = g * x.d2[k];
        r.d12[k] = g * x.d12[k] - 0.5 * g / x.v * x.d1 * x.d2[k];
    }
    return r;
}
// Dual2.pos (ad.py:230-232)
template <int NO>
AM_HD D2T<NO> dpos(const D2T<NO>& x) {
    const double gate = x.v > 0.0 ? 1.0 : 0.0;
    D2T<NO> r;
    r.v = x.v * gate;
    r.d1 = x.d1 * gate;
    for (int k = 0; k < NO; ++k) {
        r.d2[k] = x.d2[k] * gate;
        r.d12[k] = x.d12[k] * gate;
    }
    return r;
}

}  // namespace am
