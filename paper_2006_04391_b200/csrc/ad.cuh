// ad.cuh -- expression-level reverse-mode AD over sparse forward duals.
//
// Device-side equivalent of the reference's AD core (gsmkit/ad.py):
//
//  * D<M>   forward dual (ad.py:46-131 Dual1): a primal value plus tangent
//           components for the directions whose bits are set in the
//           compile-time mask M.  Directions that are structurally zero are
//           not stored and cost nothing: the mask of a result is the union
//           of its operands' masks, so sparsity of the seeds (identity
//           directions) survives through every operation without relying on
//           the compiler to fold 0*x (which IEEE forbids).  D<0> is a plain
//           double.
//  * Leaf<I,P>, Cst<P>, Add, Sub, Mul, Div, Neg, Pow, Sqrt, Exp, Log, Pos,
//           Abs: reverse expression nodes (ad.py:247-517).  Operator
//           overloading builds a compile-time tree (the "tape" is the type,
//           values live in registers); v() recomputes a subtree (ad.py:361+),
//           adj<I>(node, bv) returns the adjoint contribution reaching leaf I
//           (the sum that RLeaf.back accumulates, ad.py:339-340).  Cst drops
//           adjoints (ad.py:357-358): mixed-order expressions never
//           propagate derivatives into constant arguments.
//  * Tangent-over-adjoint (ad.py:571-617, gsm.py:494-551): the payloads of
//           a reverse sweep are D<M> values, so one sweep yields gradients
//           and directional second derivatives together.
//
// Recomputation instead of taping follows the paper: after
// inlining every v() call is a pure expression of register values and the
// compiler's value numbering shares the repeated subexpressions.
// Everything is __host__ __device__ so the same headers compile with g++.
#pragma once

#include <cmath>
#include <cstdint>
#include <type_traits>
#include <utility>

#ifdef __CUDACC__
#define AM_HD __host__ __device__ __forceinline__
#else
#define AM_HD inline
#endif

namespace am {

constexpr int kMaxDir = 16;

constexpr int popc(uint32_t m) { return m ? int(m & 1u) + popc(m >> 1) : 0; }
constexpr int slot(uint32_t m, int k) { return popc(m & ((1u << k) - 1u)); }
constexpr bool bit(uint32_t m, int k) { return (m >> k) & 1u; }

// compile-time loop: f(std::integral_constant<int, 0..N-1>)
template <class F, int... I>
AM_HD void sfor_impl(F&& f, std::integer_sequence<int, I...>) {
    (f(std::integral_constant<int, I>{}), ...);
}
template <int N, class F>
AM_HD void sfor(F&& f) {
    sfor_impl(f, std::make_integer_sequence<int, N>{});
}

// ---------------------------------------------------------------- Tup
// Minimal heterogeneous tuple usable in device code (component lists of
// payloads / nodes, like the reference's Python lists of scalar-likes).
template <int I, class T>
struct TupElem { T x; };
template <class Seq, class... T>
struct TupImpl;
template <int... I, class... T>
struct TupImpl<std::integer_sequence<int, I...>, T...> : TupElem<I, T>... {};
template <class... T>
struct Tup : TupImpl<std::make_integer_sequence<int, sizeof...(T)>, T...> {
    static constexpr int size = sizeof...(T);
};
template <int I, class T>
AM_HD T& get(TupElem<I, T>& t) { return t.x; }
template <int I, class T>
AM_HD const T& get(const TupElem<I, T>& t) { return t.x; }
template <int... I, class... T>
AM_HD Tup<T...> tup_impl(std::integer_sequence<int, I...>, const T&... x) {
    Tup<T...> r;
    ((get<I>(r) = x), ...);
    return r;
}
template <class... T>
AM_HD Tup<T...> tup(const T&... x) {
    return tup_impl(std::make_integer_sequence<int, sizeof...(T)>{}, x...);
}

// ---------------------------------------------------------------- D<M>
template <uint32_t M>
struct D {
    static constexpr uint32_t mask = M;
    static constexpr int W = popc(M);
    double v;
    double d[W > 0 ? W : 1];

    template <int k>
    AM_HD double dir() const {
        if constexpr (bit(M, k)) return d[slot(M, k)];
        else return 0.0;
    }
};

template <class T>
struct is_dual : std::false_type {};
template <uint32_t M>
struct is_dual<D<M>> : std::true_type {};

AM_HD D<0> plain(double v) { D<0> r; r.v = v; return r; }

template <int k>
AM_HD D<(1u << k)> seed(double v, double s = 1.0) {
    D<(1u << k)> r; r.v = v; r.d[0] = s; return r;
}

// elementwise tangent combination helper over the union mask
template <uint32_t A, uint32_t B, class Both, class OnlyA, class OnlyB>
AM_HD void combine(D<A | B>& r, const D<A>& x, const D<B>& y, Both both, OnlyA oa, OnlyB ob) {
    sfor<kMaxDir>([&](auto K) {
        constexpr int k = decltype(K)::value;
        if constexpr (bit(A | B, k)) {
            constexpr int ir = slot(A | B, k);
            if constexpr (bit(A, k) && bit(B, k)) r.d[ir] = both(x.d[slot(A, k)], y.d[slot(B, k)]);
            else if constexpr (bit(A, k)) r.d[ir] = oa(x.d[slot(A, k)]);
            else r.d[ir] = ob(y.d[slot(B, k)]);
        }
    });
}

template <uint32_t M, class F>
AM_HD D<M> map_d(const D<M>& x, double v, F f) {
    D<M> r; r.v = v;
    sfor<M ? D<M>::W : 0>([&](auto K) { r.d[decltype(K)::value] = f(x.d[decltype(K)::value]); });
    return r;
}

// Dual1.__add__ (ad.py:64-69)
template <uint32_t A, uint32_t B>
AM_HD D<A | B> operator+(const D<A>& x, const D<B>& y) {
    D<A | B> r; r.v = x.v + y.v;
    combine<A, B>(r, x, y, [](double p, double q) { return p + q; }, [](double p) { return p; },
                  [](double q) { return q; });
    return r;
}
// Dual1.__sub__ / __rsub__ (ad.py:71-79)
template <uint32_t A, uint32_t B>
AM_HD D<A | B> operator-(const D<A>& x, const D<B>& y) {
    D<A | B> r; r.v = x.v - y.v;
    combine<A, B>(r, x, y, [](double p, double q) { return p - q; }, [](double p) { return p; },
                  [](double q) { return -q; });
    return r;
}
// Dual1.__mul__ (ad.py:81-86): dot*o.val + val*o.dot
template <uint32_t A, uint32_t B>
AM_HD D<A | B> operator*(const D<A>& x, const D<B>& y) {
    D<A | B> r; r.v = x.v * y.v;
    const double xv = x.v, yv = y.v;
    combine<A, B>(r, x, y, [=](double p, double q) { return p * yv + xv * q; },
                  [=](double p) { return p * yv; }, [=](double q) { return q * xv; });
    return r;
}
// Dual1.__truediv__ / __rtruediv__ (ad.py:88-97)
template <uint32_t A, uint32_t B>
AM_HD D<A | B> operator/(const D<A>& x, const D<B>& y) {
    D<A | B> r;
    if constexpr (B == 0) {
        r.v = x.v / y.v;
        const double yv = y.v;
        combine<A, B>(r, x, y, [](double p, double) { return p; }, [=](double p) { return p / yv; },
                      [](double q) { return q; });
    } else {
        const double inv = 1.0 / y.v;
        const double xv = x.v;
        r.v = xv * inv;
        combine<A, B>(r, x, y, [=](double p, double q) { return (p - xv * inv * q) * inv; },
                      [=](double p) { return p * inv; }, [=](double q) { return -xv * inv * inv * q; });
    }
    return r;
}
template <uint32_t A>
AM_HD D<A> operator-(const D<A>& x) {
    return map_d(x, -x.v, [](double p) { return -p; });
}

// Dual1.__pow__ (ad.py:99-100) with a real constant exponent
template <uint32_t A>
AM_HD D<A> dpow(const D<A>& x, double c) {
    const double f = c * ::pow(x.v, c - 1.0);
    return map_d(x, ::pow(x.v, c), [=](double p) { return f * p; });
}
// Value and local partial of a constant-exponent power node as duals:
// val = x^c (dual), dval = c * x^(c-1) (dual, i.e. including c(c-1)x^(c-2)dx).
// One x^(c-2) yields all three powers (x^(c-1) = x^(c-2)*x, x^c =
// x^(c-1)*x) whenever that is exact in the limit: x > 0, or c >= 2 (x = 0
// gives 0^(c-2) in {0, 1} and zero higher powers).  Otherwise the powers are
// taken separately like Dual1.__pow__ (ad.py:99-100).
template <uint32_t A>
AM_HD void powjet(const D<A>& x, double c, D<A>& val, D<A>& dval) {
    double p0, p1, p2;
    if (x.v > 0.0) {
#ifdef AM_EXACT_POW
        p2 = ::pow(x.v, c - 2.0);
#else
        // exp((c-2) log x): a third of pow()'s instructions (pow evaluates
        // the logarithm in double-double); relative error ~|c ln x| ulp,
        // i.e. <= 1e-14 for the overstress ratios of the Norton law
        p2 = ::exp((c - 2.0) * ::log(x.v));
#endif
        p1 = p2 * x.v;
        p0 = p1 * x.v;
    } else if (c >= 2.0) {
        p2 = ::pow(x.v, c - 2.0);
        p1 = p2 * x.v;
        p0 = p1 * x.v;
    } else {
        p0 = ::pow(x.v, c);
        p1 = ::pow(x.v, c - 1.0);
        p2 = ::pow(x.v, c - 2.0);
    }
    const double f1 = c * p1;            // d/dx x^c
    const double f2 = c * ((c - 1.0) * p2);  // d/dx (c x^(c-1))
    val = map_d(x, p0, [=](double p) { return f1 * p; });
    dval = map_d(x, f1, [=](double p) { return f2 * p; });
}

template <uint32_t A>
AM_HD D<A> dsqrt(const D<A>& x) {
    const double s = ::sqrt(x.v);
    if constexpr (A == 0) {
        return plain(s);
    } else {
        const double g = 0.5 / s;
        return map_d(x, s, [=](double p) { return g * p; });
    }
}
template <uint32_t A>
AM_HD D<A> dexp(const D<A>& x) {
    const double e = ::exp(x.v);
    return map_d(x, e, [=](double p) { return e * p; });
}
template <uint32_t A>
AM_HD D<A> dlog(const D<A>& x) {
    const double xv = x.v;
    return map_d(x, ::log(xv), [=](double p) { return p / xv; });
}
// Dual1.pos (ad.py:113-115); derivative 0 at exactly 0; NaN propagates
template <uint32_t A>
AM_HD D<A> dpos(const D<A>& x) {
    if constexpr (A == 0) {
        return plain(x.v != x.v ? x.v : (x.v > 0.0 ? x.v : 0.0));
    } else {
        const double gate = x.v > 0.0 ? 1.0 : 0.0;
        return map_d(x, x.v * gate, [=](double p) { return p * gate; });
    }
}
AM_HD double sgn(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : (v == 0.0 ? 0.0 : v)); }
template <uint32_t A>
AM_HD D<A> dabs(const D<A>& x) {
    const double s = sgn(x.v);
    return map_d(x, x.v * s, [=](double p) { return p * s; });
}

// ---------------------------------------------------------------- structural zero
// Z is "no adjoint reached this leaf" (RLeaf.adj is None).
struct Z {};
template <class T>
AM_HD T operator+(Z, const T& y) { return y; }
template <uint32_t A>
AM_HD D<A> operator+(const D<A>& x, Z) { return x; }
AM_HD Z operator+(Z, Z) { return Z{}; }

// ---------------------------------------------------------------- reverse nodes
struct Node {};
template <class T>
constexpr bool is_node = std::is_base_of_v<Node, T>;

template <int I, class P>
struct Leaf : Node { P val; };
template <class P>
struct Cst : Node { P val; };
template <class A, class B>
struct Add : Node { A a; B b; };
template <class A, class B>
struct Sub : Node { A a; B b; };
template <class A, class B>
struct Mul : Node { A a; B b; };
template <class A, class B>
struct Div : Node { A a; B b; };
template <class A>
struct Neg : Node { A a; };
// Pow caches its primal value and local partial c*x^(c-1) (both as duals)
// at construction: one pow() serves v() and back() (see powjet).
template <class A, class VT>
struct Pow : Node { A a; double c; VT val, dval; };
template <class A>
struct Sqrt : Node { A a; };
template <class A>
struct Exp : Node { A a; };
template <class A>
struct Log : Node { A a; };
template <class A>
struct Pos : Node { A a; };
template <class A>
struct Abs : Node { A a; };

template <int I, class P>
AM_HD Leaf<I, P> leaf(const P& p) { Leaf<I, P> n; n.val = p; return n; }
template <class P>
AM_HD Cst<P> cst(const P& p) { Cst<P> n; n.val = p; return n; }
AM_HD Cst<D<0>> cst(double p) { return cst(plain(p)); }

// _wrap (ad.py:243-244): scalars become constants
template <class T>
AM_HD auto wrap(const T& x) {
    if constexpr (is_node<T>) return x;
    else if constexpr (is_dual<T>::value) return cst(x);
    else return cst(double(x));
}

#define AM_BIN(OP, NODE)                                                                        \
    template <class A, class B, std::enable_if_t<is_node<A> || is_node<B>, int> = 0>            \
    AM_HD auto operator OP(const A& a, const B& b) {                                            \
        using WA = decltype(wrap(a));                                                           \
        using WB = decltype(wrap(b));                                                           \
        NODE<WA, WB> n; n.a = wrap(a); n.b = wrap(b); return n;                                 \
    }
AM_BIN(+, Add)
AM_BIN(-, Sub)
AM_BIN(*, Mul)
AM_BIN(/, Div)
#undef AM_BIN

template <class A, std::enable_if_t<is_node<A>, int> = 0>
AM_HD Neg<A> operator-(const A& a) { Neg<A> n; n.a = a; return n; }
template <class A, std::enable_if_t<is_node<A>, int> = 0>
AM_HD auto npow(const A& a, double c) {
    using VT = std::decay_t<decltype(v(a))>;
    Pow<A, VT> n; n.a = a; n.c = c;
    powjet(v(a), c, n.val, n.dval);
    return n;
}
#define AM_UN(fn, NODE) \
    template <class A, std::enable_if_t<is_node<A>, int> = 0> AM_HD NODE<A> fn(const A& a) { NODE<A> n; n.a = a; return n; }
AM_UN(nsqrt, Sqrt)
AM_UN(nexp, Exp)
AM_UN(nlog, Log)
AM_UN(npos, Pos)
AM_UN(nabs, Abs)
#undef AM_UN

// ---------------------------------------------------------------- v()
template <int I, class P>
AM_HD const P& v(const Leaf<I, P>& n) { return n.val; }
template <class P>
AM_HD const P& v(const Cst<P>& n) { return n.val; }
template <class A, class B>
AM_HD auto v(const Add<A, B>& n) { return v(n.a) + v(n.b); }
template <class A, class B>
AM_HD auto v(const Sub<A, B>& n) { return v(n.a) - v(n.b); }
template <class A, class B>
AM_HD auto v(const Mul<A, B>& n) { return v(n.a) * v(n.b); }
template <class A, class B>
AM_HD auto v(const Div<A, B>& n) { return v(n.a) / v(n.b); }
template <class A>
AM_HD auto v(const Neg<A>& n) { return -v(n.a); }
template <class A, class VT>
AM_HD const VT& v(const Pow<A, VT>& n) { return n.val; }
template <class A>
AM_HD auto v(const Sqrt<A>& n) { return dsqrt(v(n.a)); }
template <class A>
AM_HD auto v(const Exp<A>& n) { return dexp(v(n.a)); }
template <class A>
AM_HD auto v(const Log<A>& n) { return dlog(v(n.a)); }
template <class A>
AM_HD auto v(const Pos<A>& n) { return dpos(v(n.a)); }
template <class A>
AM_HD auto v(const Abs<A>& n) { return dabs(v(n.a)); }

// ---------------------------------------------------------------- has<I>
template <int I, class N>
struct has : std::false_type {};
template <int I, class P>
struct has<I, Leaf<I, P>> : std::true_type {};
template <int I, class A, class B>
struct has<I, Add<A, B>> : std::bool_constant<has<I, A>::value || has<I, B>::value> {};
template <int I, class A, class B>
struct has<I, Sub<A, B>> : std::bool_constant<has<I, A>::value || has<I, B>::value> {};
template <int I, class A, class B>
struct has<I, Mul<A, B>> : std::bool_constant<has<I, A>::value || has<I, B>::value> {};
template <int I, class A, class B>
struct has<I, Div<A, B>> : std::bool_constant<has<I, A>::value || has<I, B>::value> {};
template <int I, class A>
struct has<I, Neg<A>> : has<I, A> {};
template <int I, class A, class VT>
struct has<I, Pow<A, VT>> : has<I, A> {};
template <int I, class A>
struct has<I, Sqrt<A>> : has<I, A> {};
template <int I, class A>
struct has<I, Exp<A>> : has<I, A> {};
template <int I, class A>
struct has<I, Log<A>> : has<I, A> {};
template <int I, class A>
struct has<I, Pos<A>> : has<I, A> {};
template <int I, class A>
struct has<I, Abs<A>> : has<I, A> {};

// ---------------------------------------------------------------- adj<I>()
// Contribution of subtree n to the adjoint of leaf I given the incoming
// adjoint bv (the back() rules of ad.py:361-517).  Subtrees that do not
// contain leaf I are pruned at compile time; the incoming adjoint of a
// child is built lazily so pruned branches generate no code.
template <int I, class N, class F>
AM_HD auto adjl(const N& n, F&& mk);

template <int I, int J, class P, class BV>
AM_HD auto adj(const Leaf<J, P>&, const BV& bv) {
    if constexpr (I == J) return bv;
    else return Z{};
}
template <int I, class P, class BV>
AM_HD Z adj(const Cst<P>&, const BV&) { return Z{}; }
template <int I, class A, class B, class BV>
AM_HD auto adj(const Add<A, B>& n, const BV& bv) {
    return adjl<I>(n.a, [&] { return bv; }) + adjl<I>(n.b, [&] { return bv; });
}
template <int I, class A, class B, class BV>
AM_HD auto adj(const Sub<A, B>& n, const BV& bv) {
    return adjl<I>(n.a, [&] { return bv; }) + adjl<I>(n.b, [&] { return -bv; });
}
template <int I, class A, class B, class BV>
AM_HD auto adj(const Mul<A, B>& n, const BV& bv) {
    return adjl<I>(n.a, [&] { return bv * v(n.b); }) + adjl<I>(n.b, [&] { return bv * v(n.a); });
}
template <int I, class A, class B, class BV>
AM_HD auto adj(const Div<A, B>& n, const BV& bv) {
    return adjl<I>(n.a, [&] { return bv / v(n.b); }) + adjl<I>(n.b, [&] {
               const auto bval = v(n.b);
               return (-bv * v(n.a)) / (bval * bval);
           });
}
template <int I, class A, class BV>
AM_HD auto adj(const Neg<A>& n, const BV& bv) { return adjl<I>(n.a, [&] { return -bv; }); }
// RPow.back: bv * (c * av**(c-1)), the partial cached by powjet
template <int I, class A, class VT, class BV>
AM_HD auto adj(const Pow<A, VT>& n, const BV& bv) {
    return adjl<I>(n.a, [&] { return bv * n.dval; });
}
// RSqrt.back: bv * (0.5 / sqrt(av))
template <int I, class A, class BV>
AM_HD auto adj(const Sqrt<A>& n, const BV& bv) {
    return adjl<I>(n.a, [&] { return bv * (plain(0.5) / dsqrt(v(n.a))); });
}
template <int I, class A, class BV>
AM_HD auto adj(const Exp<A>& n, const BV& bv) { return adjl<I>(n.a, [&] { return bv * dexp(v(n.a)); }); }
template <int I, class A, class BV>
AM_HD auto adj(const Log<A>& n, const BV& bv) { return adjl<I>(n.a, [&] { return bv / v(n.a); }); }
// RPos.back: gate on the primal (ad.py:502-504)
template <int I, class A, class BV>
AM_HD auto adj(const Pos<A>& n, const BV& bv) {
    return adjl<I>(n.a, [&] { return bv * plain(v(n.a).v > 0.0 ? 1.0 : 0.0); });
}
template <int I, class A, class BV>
AM_HD auto adj(const Abs<A>& n, const BV& bv) { return adjl<I>(n.a, [&] { return bv * plain(sgn(v(n.a).v)); }); }

template <int I, class N, class F>
AM_HD auto adjl(const N& n, F&& mk) {
    if constexpr (has<I, N>::value) return adj<I>(n, mk());
    else return Z{};
}

// RLeaf.adjoint (ad.py:342-343): value*0.0 when nothing reached the leaf
template <class T, class P>
AM_HD auto adjoint_or_zero(const T& a, const P& leafval) {
    if constexpr (std::is_same_v<T, Z>) return leafval * plain(0.0);
    else return a;
}

// grad of root w.r.t. leaf I with seed bv (grad_reverse, ad.py:555-568)
template <int I, class Root, class P>
AM_HD auto gradient(const Root& root, const P& leafval, double seed = 1.0) {
    return adjoint_or_zero(adj<I>(root, plain(seed)), leafval);
}

}  // namespace am
