// em_jvp.cuh — forward-mode derivatives of the path coefficient with respect to
// device positions and orientations.
//
// With tracked positions the reference re-derives the geometry by closed-form
// mirroring across the frozen interaction planes (geometry_for_positions,
// em.py:258-282) and evaluates the transfer (em.py:291-312) on tape scalars.
// Here the same arithmetic runs on a one-tangent dual number; a launch
// evaluates every (path, tx slant, tangent) with tangents
//   0-2 tx position, 3-5 rx position, 6-8 tx (yaw, pitch, roll), 9-11 rx ypr,
// so the Jacobian column of a[p, s, r] w.r.t. each parameter comes out of one
// thread.  PyTorch's backward contracts it with the upstream gradient.
// Branches (dipole null, tr38901 floors, csqrt_posreal guards, normal-
// incidence axis) follow the reference's value-based decisions, i.e. the
// tape's subgradients.
#pragma once
#include "em.cuh"

namespace rt {

constexpr int NJ = 12;

struct D1 {
    double v, d;
};
__device__ inline D1 dc(double v) { return D1{v, 0.0}; }
__device__ inline D1 operator+(D1 a, D1 b) { return D1{a.v + b.v, a.d + b.d}; }
__device__ inline D1 operator-(D1 a, D1 b) { return D1{a.v - b.v, a.d - b.d}; }
__device__ inline D1 operator-(D1 a) { return D1{-a.v, -a.d}; }
__device__ inline D1 operator*(D1 a, D1 b) { return D1{a.v * b.v, a.d * b.v + a.v * b.d}; }
__device__ inline D1 operator*(D1 a, double s) { return D1{a.v * s, a.d * s}; }
__device__ inline D1 operator*(double s, D1 a) { return D1{s * a.v, s * a.d}; }
__device__ inline D1 operator/(D1 a, D1 b) {
    double inv = 1.0 / b.v;
    return D1{a.v / b.v, a.d * inv - a.v * inv * inv * b.d};
}
__device__ inline D1 operator/(D1 a, double s) { return D1{a.v / s, a.d / s}; }
__device__ inline D1 operator/(double s, D1 b) {
    double inv = 1.0 / b.v;
    return D1{s / b.v, -s * inv * inv * b.d};
}
__device__ inline D1 operator+(D1 a, double s) { return D1{a.v + s, a.d}; }
__device__ inline D1 operator-(D1 a, double s) { return D1{a.v - s, a.d}; }
__device__ inline D1 operator-(double s, D1 a) { return D1{s - a.v, -a.d}; }
__device__ inline D1 dsqrt(D1 a) {
    double v = sqrt(a.v);
    return D1{v, v != 0.0 ? a.d * (0.5 / v) : 0.0};
}
__device__ inline D1 dsin(D1 a) { return D1{sin(a.v), a.d * cos(a.v)}; }
__device__ inline D1 dcos(D1 a) { return D1{cos(a.v), -a.d * sin(a.v)}; }
__device__ inline D1 dexp(D1 a) {
    double v = exp(a.v);
    return D1{v, a.d * v};
}
__device__ inline D1 datan2(D1 y, D1 x) {
    double q = y.v * y.v + x.v * x.v;
    return D1{atan2(y.v, x.v), q != 0.0 ? (x.v * y.d - y.v * x.d) / q : 0.0};
}

struct V1 {
    D1 x, y, z;
};
__device__ inline V1 vsub(V1 a, V1 b) { return V1{a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ inline D1 vdot(V1 a, V1 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }   // t_dot
__device__ inline D1 vdot(V1 a, d3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ inline V1 vcross(V1 a, V1 b) {
    return V1{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ inline V1 vcross(V1 a, d3 b) {
    return V1{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ inline V1 vnormalize(V1 a) {   // t_normalize
    D1 n = dsqrt(vdot(a, a));
    return V1{a.x / n, a.y / n, a.z / n};
}

struct CD {
    D1 re, im;
};
__device__ inline CD cdm(CD a, CD b) { return CD{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
__device__ inline CD cdd(CD a, CD o) {
    D1 d = o.re * o.re + o.im * o.im;
    return CD{(a.re * o.re + a.im * o.im) / d, (a.im * o.re - a.re * o.im) / d};
}
__device__ inline CD cds(CD a, D1 s) { return CD{a.re * s, a.im * s}; }
__device__ inline CD cda(CD a, CD b) { return CD{a.re + b.re, a.im + b.im}; }
__device__ inline CD cdsub(CD a, CD b) { return CD{a.re - b.re, a.im - b.im}; }

// geometry.py:50-59
__device__ inline void rot_rows(D1 yaw, D1 pitch, D1 roll, D1* R) {
    D1 cy = dcos(yaw), sy = dsin(yaw), cp = dcos(pitch), sp = dsin(pitch);
    D1 cr = dcos(roll), sr = dsin(roll);
    R[0] = cy * cp; R[1] = cy * sp * sr - sy * cr; R[2] = cy * sp * cr + sy * sr;
    R[3] = sy * cp; R[4] = sy * sp * sr + cy * cr; R[5] = sy * sp * cr - cy * sr;
    R[6] = -sp; R[7] = cp * sr; R[8] = cp * cr;
}

__device__ inline void pattern_d(int id, D1 theta, D1 phi, D1& eth, D1& eph) {   // em.py:42-75
    eth = dc(0.0);
    eph = dc(0.0);
    if (id == 0 || id == 3) {
        eth = dc(1.0);
    } else if (id == 1) {
        D1 s = dsin(theta);
        if (s.v < 1e-9) return;
        eth = sqrt(1.643) * dcos(1.5707963267948966 * dcos(theta)) / s;
    } else if (id == 2) {
        const double deg = 180.0 / PI;
        D1 tilt = theta * deg - 90.0, pan = phi * deg;
        D1 av = 12.0 * (tilt / 65.0) * (tilt / 65.0);
        if (!(av.v <= 30.0)) av = dc(30.0);
        D1 ah = 12.0 * (pan / 65.0) * (pan / 65.0);
        if (!(ah.v <= 30.0)) ah = dc(30.0);
        D1 s = av + ah;
        if (!(s.v <= 30.0)) s = dc(30.0);
        eth = dexp((8.0 - s) * (2.302585092994046 / 20.0));
    } else if (id == 4) {
        eph = dc(1.0);
    }
}

__device__ inline V1 element_field_d(int pat, double slant, const D1* R, V1 k) {   // em.py:98-118
    V1 kb = V1{R[0] * k.x + R[3] * k.y + R[6] * k.z, R[1] * k.x + R[4] * k.y + R[7] * k.z,
               R[2] * k.x + R[5] * k.y + R[8] * k.z};
    double cz = cos(slant), sz = sin(slant);
    V1 ke = V1{kb.x, cz * kb.y + sz * kb.z, -sz * kb.y + cz * kb.z};
    D1 theta = datan2(dsqrt(ke.x * ke.x + ke.y * ke.y), ke.z);
    D1 phi = datan2(ke.y, ke.x);
    D1 eth, eph;
    pattern_d(pat, theta, phi, eth, eph);
    D1 ct = dcos(theta), st = dsin(theta), cp = dcos(phi), sp = dsin(phi);
    V1 ee = V1{eth * (ct * cp) + eph * (-sp), eth * (ct * sp) + eph * cp, eth * (-st)};
    V1 eb = V1{ee.x, cz * ee.y - sz * ee.z, sz * ee.y + cz * ee.z};
    return V1{R[0] * eb.x + R[1] * eb.y + R[2] * eb.z, R[3] * eb.x + R[4] * eb.y + R[5] * eb.z,
              R[6] * eb.x + R[7] * eb.y + R[8] * eb.z};
}

__device__ inline CD csqrt_posreal_d(CD z) {   // autodiff.py:365-382
    D1 m = dsqrt(z.re * z.re + z.im * z.im);
    D1 u2 = (m + z.re) * 0.5, v2 = (m - z.re) * 0.5;
    D1 u = u2.v > 0.0 ? dsqrt(u2) : u2 * 0.0;
    D1 v = v2.v > 0.0 ? dsqrt(v2) : v2 * 0.0;
    if (z.im.v < 0.0) v = -v;
    return CD{u, v};
}

__device__ inline void fresnel_d(c2 eta, D1 ci, CD& rte, CD& rtm) {   // em.py:123-141
    D1 sin2 = 1.0 - ci * ci;
    CD w = csqrt_posreal_d(CD{dc(eta.re) - sin2, dc(eta.im)});
    CD c = CD{ci, dc(0.0)};
    rte = cdd(cdsub(c, w), cda(c, w));
    CD ec = CD{eta.re * ci, eta.im * ci};
    rtm = cdd(cdsub(w, ec), cda(w, ec));
}

struct F3 {
    CD x, y, z;
};
__device__ inline CD fdot(const F3& f, V1 e) {
    return cda(cda(cds(f.x, e.x), cds(f.y, e.y)), cds(f.z, e.z));
}

__device__ inline void reflect_d(F3& f, V1 kin, V1 kout, d3 n, CD rte, CD rtm) {   // em.py:144-171
    V1 e = vcross(kin, n);
    if (vdot(e, e).v < 1e-16) {
        double a0 = fabs(kin.x.v), a1 = fabs(kin.y.v), a2 = fabs(kin.z.v);
        d3 axis = d3{1.0, 0.0, 0.0};
        double mn = a0;
        if (a1 < mn) { mn = a1; axis = d3{0.0, 1.0, 0.0}; }
        if (a2 < mn) { axis = d3{0.0, 0.0, 1.0}; }
        e = vcross(kin, axis);
    }
    e = vnormalize(e);
    V1 epi = vcross(kin, e), epr = vcross(e, kout);
    CD fp = fdot(f, e), fa = fdot(f, epi);
    CD gp = cdm(rte, fp), ga = cdm(rtm, fa);
    f.x = cda(cds(gp, e.x), cds(ga, epr.x));
    f.y = cda(cds(gp, e.y), cds(ga, epr.y));
    f.z = cda(cds(gp, e.z), cds(ga, epr.z));
}

struct JvpArgs {
    long long n;
    int L;
    const signed char* order;
    const int* seq;
    const double* verts;   // the traced path: planes are fixed through its vertices
    const double* nrm;     // oriented normals
    const double* tx_pos;  // [P*3]
    const double* rx_pos;
    const double* tx_ypr;
    const double* rx_ypr;
    int tx_pat, rx_pat;
    const double* tx_slants;
    int n_st;
    const double* rx_slants;
    int n_sr;
    const double* eta;
    const int* prim_mat;
    double wavelength, frequency;
};

// a[p, s, r] (value) and d a / d theta_w for tangent w: one thread per (p, s, w)
__global__ void k_transfer_jvp(const __grid_constant__ JvpArgs A, double* a_out /*[P*S*R*2]*/,
                               double* jac /*[P*S*R*NJ*2]*/) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= A.n * A.n_st * NJ) return;
    int w = (int)(i % NJ);
    long long ps = i / NJ;
    long long p = ps / A.n_st;
    int s = (int)(ps - p * A.n_st);
    int K = A.order[p];
    auto seeded = [&](const double* src, int base) {
        V1 v{dc(src[3 * p]), dc(src[3 * p + 1]), dc(src[3 * p + 2])};
        if (w == base) v.x.d = 1.0;
        if (w == base + 1) v.y.d = 1.0;
        if (w == base + 2) v.z.d = 1.0;
        return v;
    };
    V1 tx = seeded(A.tx_pos, 0), rx = seeded(A.rx_pos, 3);
    V1 to = seeded(A.tx_ypr, 6), ro = seeded(A.rx_ypr, 9);
    D1 Rt[9], Rr[9];
    rot_rows(to.x, to.y, to.z, Rt);
    rot_rows(ro.x, ro.y, ro.z, Rr);
    // geometry_for_positions: planes through the traced vertices, closed-form mirror solve
    const double* vp = A.verts + p * (A.L + 2) * 3;
    const double* np_ = A.nrm + p * A.L * 3;
    d3 nk[MAX_DEPTH];
    double ck[MAX_DEPTH];
    for (int j = 0; j < K; ++j) {
        nk[j] = ld3(np_ + 3 * j);
        ck[j] = tdot(nk[j], ld3(vp + 3 * (j + 1)));
    }
    V1 img[MAX_DEPTH + 1];
    img[0] = tx;
    for (int j = 0; j < K; ++j) {   // _mirror (tracer.py:71-73)
        D1 kk = 2.0 * (vdot(img[j], nk[j]) - ck[j]);
        img[j + 1] = V1{img[j].x - nk[j].x * kk, img[j].y - nk[j].y * kk, img[j].z - nk[j].z * kk};
    }
    V1 pts[MAX_DEPTH];
    V1 cur = rx;
    for (int j = K - 1; j >= 0; --j) {   // solve_points back-substitution (tracer.py:90-101)
        V1 seg = vsub(img[j + 1], cur);
        D1 denom = vdot(seg, nk[j]);
        D1 sj = (ck[j] - vdot(cur, nk[j])) / denom;
        pts[j] = V1{cur.x + seg.x * sj, cur.y + seg.y * sj, cur.z + seg.z * sj};
        cur = pts[j];
    }
    V1 dir[MAX_DEPTH + 1];
    D1 length = dc(0.0);
    V1 a = tx;
    for (int j = 0; j <= K; ++j) {
        V1 b = j < K ? pts[j] : rx;
        V1 sgm = vsub(b, a);
        dir[j] = vnormalize(sgm);
        length = length + dsqrt(vdot(sgm, sgm));
        a = b;
    }
    D1 delay = length / SPEED_OF_LIGHT;
    // transfer (em.py:291-312)
    V1 ef = element_field_d(A.tx_pat, A.tx_slants[s], Rt, dir[0]);
    F3 f = F3{CD{ef.x, dc(0.0)}, CD{ef.y, dc(0.0)}, CD{ef.z, dc(0.0)}};
    for (int j = 0; j < K; ++j) {
        int m = A.prim_mat[A.seq[p * A.L + j]];
        c2 et = c2{A.eta[2 * m], A.eta[2 * m + 1]};
        D1 ci = -vdot(dir[j], nk[j]);   // geometry_for_positions cosines
        CD rte, rtm;
        fresnel_d(et, ci, rte, rtm);
        reflect_d(f, dir[j], dir[j + 1], nk[j], rte, rtm);
    }
    D1 amp = A.wavelength / (2.0 * TWO_PI * length);
    D1 phase = -TWO_PI * A.frequency * delay;
    CD ph = CD{dcos(phase), dsin(phase)};
    V1 karr = V1{dir[K].x * -1.0, dir[K].y * -1.0, dir[K].z * -1.0};
    for (int r = 0; r < A.n_sr; ++r) {
        V1 rf = element_field_d(A.rx_pat, A.rx_slants[r], Rr, karr);
        CD coup = cda(cda(cds(f.x, rf.x), cds(f.y, rf.y)), cds(f.z, rf.z));
        CD av = cdm(cds(coup, amp), ph);
        long long o = (p * A.n_st + s) * A.n_sr + r;
        jac[(o * NJ + w) * 2] = av.re.d;
        jac[(o * NJ + w) * 2 + 1] = av.im.d;
        if (w == 0) {
            a_out[2 * o] = av.re.v;
            a_out[2 * o + 1] = av.im.v;
        }
    }
}

}  // namespace rt
