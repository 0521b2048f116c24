// fasmg_natural.cu -- the reference kernel ABI on device arrays in the
// reference (natural) layout, plus ghost fill and numpy-ordered reductions.
//
// These are the drop-in replacements for the 16 names dispatched by
// KER/__init__.py:37-46 (signatures of KER/numpy_backend.py), taking device
// pointers to core views with element strides.  The fast FAS V-cycle does
// not use them (it runs on the parity-blocked layout, fasmg_engine.cu); they
// back the field-level API (smooth, residual, restrict, ... on Field
// objects) and the WENO / staggered operators of the projection drivers.
#include <string.h>

#include "fasmg_common.cuh"
#include "fasmg_internal.h"

namespace fasmg {

#define I2(s, i, j) ((long)(i) * (s)[0] + (long)(j) * (s)[1])
#define I3(s, i, j, k) ((long)(i) * (s)[0] + (long)(j) * (s)[1] + (long)(k) * (s)[2])

struct S3 { long s[3]; };

static inline S3 mk(const long* st) { S3 r; r.s[0] = st[0]; r.s[1] = st[1]; r.s[2] = st[2]; return r; }

static inline int nblk(long n, int t) { return (int)((n + t - 1) / t); }
static constexpr int TPB = 256;

// ---------------------------------------------------------------- GS sweeps
// KER/numpy_backend.py:27-62: p = (h2*f + b*nsum)/denom, nsum in E,W,N,S,T,B
__global__ void k_gs2(double* p, S3 ps, const double* f, S3 fs, double b, double h2,
                      double denom, int i0, int j0, int ni, int nj) {
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (t >= (long)ni * nj) return;
    int i = i0 + 2 * (int)(t / nj), j = j0 + 2 * (int)(t % nj);
    double nsum = ad(ad(ad(p[I2(ps.s, i + 1, j)], p[I2(ps.s, i - 1, j)]), p[I2(ps.s, i, j + 1)]),
                     p[I2(ps.s, i, j - 1)]);
    p[I2(ps.s, i, j)] = dv(ad(ml(h2, f[I2(fs.s, i, j)]), ml(b, nsum)), denom);
}

__global__ void k_gs3(double* p, S3 ps, const double* f, S3 fs, double b, double h2,
                      double denom, int i0, int j0, int k0, int ni, int nj, int nk) {
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (t >= (long)ni * nj * nk) return;
    int k = k0 + 2 * (int)(t % nk);
    long r = t / nk;
    int j = j0 + 2 * (int)(r % nj), i = i0 + 2 * (int)(r / nj);
    double nsum = ad(ad(ad(ad(ad(p[I3(ps.s, i + 1, j, k)], p[I3(ps.s, i - 1, j, k)]),
                                 p[I3(ps.s, i, j + 1, k)]), p[I3(ps.s, i, j - 1, k)]),
                           p[I3(ps.s, i, j, k + 1)]), p[I3(ps.s, i, j, k - 1)]);
    p[I3(ps.s, i, j, k)] = dv(ad(ml(h2, f[I3(fs.s, i, j, k)]), ml(b, nsum)), denom);
}

static inline int prng(int lo, int par) { return lo + ((par - lo) & 1); }

// ----------------------------------------------------- apply_op / residual
// KER/numpy_backend.py:69-112
template <bool RES>
__global__ void k_op2(double* out, S3 os, const double* p, S3 ps, const double* fsrc, S3 fs,
                      double a, double b, double inv_h2, int ilo, int jlo, int ni, int nj) {
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (t >= (long)ni * nj) return;
    int i = ilo + (int)(t / nj), j = jlo + (int)(t % nj);
    double c = p[I2(ps.s, i, j)];
    double nsum = ad(ad(ad(p[I2(ps.s, i + 1, j)], p[I2(ps.s, i - 1, j)]), p[I2(ps.s, i, j + 1)]),
                     p[I2(ps.s, i, j - 1)]);
    double lap = ml(sb(nsum, ml(4.0, c)), inv_h2);
    double op = sb(ml(a, c), ml(b, lap));
    out[I2(os.s, i, j)] = RES ? sb(fsrc[I2(fs.s, i, j)], op) : op;
}

template <bool RES>
__global__ void k_op3(double* out, S3 os, const double* p, S3 ps, const double* fsrc, S3 fs,
                      double a, double b, double inv_h2, int ilo, int jlo, int klo, int ni,
                      int nj, int nk) {
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (t >= (long)ni * nj * nk) return;
    int k = klo + (int)(t % nk);
    long r = t / nk;
    int j = jlo + (int)(r % nj), i = ilo + (int)(r / nj);
    double c = p[I3(ps.s, i, j, k)];
    double nsum = ad(ad(ad(ad(ad(p[I3(ps.s, i + 1, j, k)], p[I3(ps.s, i - 1, j, k)]),
                                 p[I3(ps.s, i, j + 1, k)]), p[I3(ps.s, i, j - 1, k)]),
                           p[I3(ps.s, i, j, k + 1)]), p[I3(ps.s, i, j, k - 1)]);
    double lap = ml(sb(nsum, ml(6.0, c)), inv_h2);
    double op = sb(ml(a, c), ml(b, lap));
    out[I3(os.s, i, j, k)] = RES ? sb(fsrc[I3(fs.s, i, j, k)], op) : op;
}

// -------------------------------------------------- cell-centered transfers
// KER/numpy_backend.py:119-155 (3D add order: numba :238-253)
__global__ void k_rcc2(const double* fn, S3 fs, double* co, S3 cs, int m0, int n0) {
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (t >= (long)m0 * n0) return;
    int i = 1 + (int)(t / n0), j = 1 + (int)(t % n0);
    int fi = 2 * i, fj = 2 * j;
    double acc = ad(ad(ad(fn[I2(fs.s, fi - 1, fj - 1)], fn[I2(fs.s, fi - 1, fj)]),
                       fn[I2(fs.s, fi, fj - 1)]), fn[I2(fs.s, fi, fj)]);
    co[I2(cs.s, i, j)] = ml(acc, 0.25);
}

__global__ void k_rcc3(const double* fn, S3 fs, double* co, S3 cs, int m0, int n0, int l0) {
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (t >= (long)m0 * n0 * l0) return;
    int k = 1 + (int)(t % l0);
    long r = t / l0;
    int j = 1 + (int)(r % n0), i = 1 + (int)(r / n0);
    int fi = 2 * i, fj = 2 * j, fk = 2 * k;
    double acc = fn[I3(fs.s, fi - 1, fj - 1, fk - 1)];
    acc = ad(acc, fn[I3(fs.s, fi - 1, fj - 1, fk)]);
    acc = ad(acc, fn[I3(fs.s, fi - 1, fj, fk - 1)]);
    acc = ad(acc, fn[I3(fs.s, fi - 1, fj, fk)]);
    acc = ad(acc, fn[I3(fs.s, fi, fj - 1, fk - 1)]);
    acc = ad(acc, fn[I3(fs.s, fi, fj - 1, fk)]);
    acc = ad(acc, fn[I3(fs.s, fi, fj, fk - 1)]);
    acc = ad(acc, fn[I3(fs.s, fi, fj, fk)]);
    co[I3(cs.s, i, j, k)] = ml(acc, 0.125);
}

__global__ void k_pcc2(const double* co, S3 cs, double* fn, S3 fs, int m0, int n0) {
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (t >= (long)m0 * n0) return;
    int i = 1 + (int)(t / n0), j = 1 + (int)(t % n0);
    int fi = 2 * i, fj = 2 * j;
    double c = co[I2(cs.s, i, j)];
    fn[I2(fs.s, fi - 1, fj - 1)] = c;
    fn[I2(fs.s, fi - 1, fj)] = c;
    fn[I2(fs.s, fi, fj - 1)] = c;
    fn[I2(fs.s, fi, fj)] = c;
}

__global__ void k_pcc3(const double* co, S3 cs, double* fn, S3 fs, int m0, int n0, int l0) {
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (t >= (long)m0 * n0 * l0) return;
    int k = 1 + (int)(t % l0);
    long r = t / l0;
    int j = 1 + (int)(r % n0), i = 1 + (int)(r / n0);
    int fi = 2 * i, fj = 2 * j, fk = 2 * k;
    double c = co[I3(cs.s, i, j, k)];
    for (int di = -1; di <= 0; ++di)
        for (int dj = -1; dj <= 0; ++dj)
            for (int dk = -1; dk <= 0; ++dk) fn[I3(fs.s, fi + di, fj + dj, fk + dk)] = c;
}

// --------------------------------------------------- edge-axis-0 transfers
// KER/numpy_backend.py:162-224
__global__ void k_red2(const double* fn, S3 fs, double* co, S3 cs, int m0, int n0) {
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (t >= (long)(m0 - 1) * n0) return;
    int i = 1 + (int)(t / n0), j = 1 + (int)(t % n0);
    int fi = 2 * i, fj = 2 * j;
    double t1 = ad(ad(fn[I2(fs.s, fi - 1, fj - 1)], ml(2.0, fn[I2(fs.s, fi - 1, fj)])),
                   fn[I2(fs.s, fi - 1, fj + 1)]);
    double t2 = ad(ad(fn[I2(fs.s, fi, fj - 1)], ml(2.0, fn[I2(fs.s, fi, fj)])),
                   fn[I2(fs.s, fi, fj + 1)]);
    co[I2(cs.s, i, j)] = ml(ad(t1, t2), 0.125);
}

__device__ __forceinline__ double red3_point(const double* fn, const S3& fs, int i, int j,
                                             int k) {
    int fi = 2 * i, fj = 2 * j, fk = 2 * k;
    double tang[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        int fx = fi - 1 + c;
        double rows[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            int fy = fj - 1 + r;
            rows[r] = ml(ad(ad(fn[I3(fs.s, fx, fy, fk - 1)], ml(2.0, fn[I3(fs.s, fx, fy, fk)])),
                            fn[I3(fs.s, fx, fy, fk + 1)]), 0.25);
        }
        tang[c] = ml(ad(ad(rows[0], ml(2.0, rows[1])), rows[2]), 0.25);
    }
    return ml(ad(tang[0], tang[1]), 0.5);
}

__global__ void k_red3(const double* fn, S3 fs, double* co, S3 cs, int m0, int n0, int l0) {
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (t >= (long)(m0 - 1) * n0 * l0) return;
    int k = 1 + (int)(t % l0);
    long r = t / l0;
    int j = 1 + (int)(r % n0), i = 1 + (int)(r / n0);
    co[I3(cs.s, i, j, k)] = red3_point(fn, fs, i, j, k);
}

__global__ void k_ped2_lines(const double* co, S3 cs, double* fn, S3 fs, int m0, int n0) {
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (t >= (long)(m0 + 1) * n0) return;
    int i = (int)(t / n0), j = 1 + (int)(t % n0);
    int fi = 2 * i, fj = 2 * j;
    double cc = co[I2(cs.s, i, j)];
    fn[I2(fs.s, fi, fj - 1)] = ml(ad(ml(3.0, cc), co[I2(cs.s, i, j - 1)]), 0.25);
    fn[I2(fs.s, fi, fj)] = ml(ad(ml(3.0, cc), co[I2(cs.s, i, j + 1)]), 0.25);
}

__global__ void k_ped2_mid(double* fn, S3 fs, int m0, int n0) {
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    long nn = 2L * n0;
    if (t >= (long)m0 * nn) return;
    int i = (int)(t / nn), fj = 1 + (int)(t % nn);
    int fi = 2 * i + 1;
    fn[I2(fs.s, fi, fj)] = ml(ad(fn[I2(fs.s, fi - 1, fj)], fn[I2(fs.s, fi + 1, fj)]), 0.5);
}

__global__ void k_ped3_lines(const double* co, S3 cs, double* fn, S3 fs, int m0, int n0,
                             int l0) {
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (t >= (long)(m0 + 1) * n0 * l0) return;
    int k = 1 + (int)(t % l0);
    long r = t / l0;
    int j = 1 + (int)(r % n0), i = (int)(r / n0);
    int fi = 2 * i, fj = 2 * j, fk = 2 * k;
#pragma unroll
    for (int dj = -1; dj <= 1; dj += 2) {
        double t_near = ml(ad(ml(3.0, co[I3(cs.s, i, j, k)]), co[I3(cs.s, i, j + dj, k)]), 0.25);
#pragma unroll
        for (int dk = -1; dk <= 1; dk += 2) {
            double t_far = ml(ad(ml(3.0, co[I3(cs.s, i, j, k + dk)]),
                                 co[I3(cs.s, i, j + dj, k + dk)]), 0.25);
            int fy = dj == -1 ? fj - 1 : fj;
            int fz = dk == -1 ? fk - 1 : fk;
            fn[I3(fs.s, fi, fy, fz)] = ml(ad(ml(3.0, t_near), t_far), 0.25);
        }
    }
}

__global__ void k_ped3_mid(double* fn, S3 fs, int m0, int n0, int l0) {
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    long nj = 2L * n0, nk = 2L * l0;
    if (t >= (long)m0 * nj * nk) return;
    int fk = 1 + (int)(t % nk);
    long r = t / nk;
    int fj = 1 + (int)(r % nj), i = (int)(r / nj);
    int fi = 2 * i + 1;
    fn[I3(fs.s, fi, fj, fk)] =
        ml(ad(fn[I3(fs.s, fi - 1, fj, fk)], fn[I3(fs.s, fi + 1, fj, fk)]), 0.5);
}

// ------------------------------------------------------------------ WENO3
// KER/numpy_backend.py:231-277 / numba :394-410
__device__ __forceinline__ double weno_point(double dm2, double dm1, double dp1, double dp2,
                                             double w, double inv_2h, double eps) {
    double c0, c1, r0, r1;
    if (w >= 0.0) {
        c0 = sb(ml(3.0, dm1), dm2);
        c1 = ad(dm1, dp1);
        r0 = sb(dm1, dm2);
        r1 = sb(dp1, dm1);
    } else {
        c0 = sb(ml(3.0, dp1), dp2);
        c1 = ad(dp1, dm1);
        r0 = sb(dp1, dp2);
        r1 = sb(dm1, dp1);
    }
    double e0 = ad(eps, ml(r0, r0));
    double e1 = ad(eps, ml(r1, r1));
    double a0 = dv(1.0 / 3.0, ml(e0, e0));
    double a1 = dv(2.0 / 3.0, ml(e1, e1));
    return ml(dv(ad(ml(a0, c0), ml(a1, c1)), ad(a0, a1)), inv_2h);
}

// The reference runs these axis-0 kernels on moveaxis views, so the view's
// last axis may be the strided one; `fast` names the view axis with the
// smallest output stride, which consecutive threads walk (coalescing only:
// every point's arithmetic is unchanged).
// Whole weno3_convect of one target component in one pass (PKG/weno.py:
// 54-91): for every target interior point, sum over derivative axes a of
// wind_a * weno3(q along a), accumulated from +0.0 in axis order exactly as
// the reference's per-axis kernel calls on a zeroed array; the wind of a
// foreign axis is the 4-point average 0.25*((v00+v01)+(v10+v11)) of
// _avg_to_target (PKG/weno.py:26-51), evaluated in place instead of being
// materialised.  vel[a]: data pointer + strides of component a (halo g),
// q = vel[target].  One thread per target interior point.
struct Vel3 { const double* p[3]; long s[3][3]; int n[3][3]; };
template <int DIM, int TGT>
__global__ void __launch_bounds__(256) k_weno_convect(double* out, S3 os, Vel3 V, int g, int e0,
                                                      int e1, int e2, double inv_2h, double eps) {
    // the thread's first point (box mapping, no 64-bit div/mod); every
    // address below is a per-thread base advanced by the axis-0 stride for
    // each further point of the z walk
    int I[3];
    if (!box_coords(DIM, e0, e1, e2, 0, I)) return;
    const double* q = V.p[TGT];
    long qc = 0;  // q at data index I + g
#pragma unroll
    for (int b = 0; b < DIM; ++b) qc += (long)(I[b] + g) * V.s[TGT][b];
    const double* qp = q + qc;
    // wind of a foreign axis a: core index of vel[a] is target axis I+1+dt,
    // own axis I+da, else I+1; data index = core + g - 1
    const double* wp[DIM];
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
        long base = 0;
#pragma unroll
        for (int b = 0; b < DIM; ++b) {
            const int c = b == TGT ? I[b] + 1 : (b == a ? I[b] : I[b] + 1);
            base += (long)(c + g - 1) * V.s[a][b];
        }
        wp[a] = V.p[a] + base;
    }
    double* op = out + I3(os.s, I[0], I[1], I[2]);
    const int nz = DIM == 3 ? min(BOX_Z, e0 - I[0]) : 1;
    for (int z = 0; z < nz; ++z) {
        // every load first (5 q values per axis, 4 wind values per foreign
        // axis), then the per-axis WENO points (independent), then the
        // ordered sum
        double qv[DIM][5], w[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            const long sa = V.s[TGT][a];
#pragma unroll
            for (int d = 0; d < 5; ++d) qv[a][d] = qp[(d - 2) * sa];
        }
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            if (a == TGT) continue;
            const long st = V.s[a][TGT], sa = V.s[a][a];
            const double* va = wp[a];
            const double v00 = va[0], v01 = va[sa], v10 = va[st], v11 = va[st + sa];
            w[a] = ml(0.25, ad(ad(v00, v01), ad(v10, v11)));  // PKG/weno.py:51
        }
        w[TGT] = qv[0][2];
        double term[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            const double dm2 = sb(qv[a][1], qv[a][0]), dm1 = sb(qv[a][2], qv[a][1]);
            const double dp1 = sb(qv[a][3], qv[a][2]), dp2 = sb(qv[a][4], qv[a][3]);
            term[a] = ml(w[a], weno_point(dm2, dm1, dp1, dp2, w[a], inv_2h, eps));
        }
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < DIM; ++a) acc = ad(acc, term[a]);
        *op = acc;
        qp += V.s[TGT][0];
#pragma unroll
        for (int a = 0; a < DIM; ++a) wp[a] += V.s[a][0];
        op += os.s[0];
    }
}

__global__ void k_weno2(double* out, S3 os, const double* q, S3 qs, const double* wind, S3 ws,
                        int ni, int nj, int oi, int oj, double inv_2h, double eps, int fast) {
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (t >= (long)ni * nj) return;
    int ii, jj;
    if (fast == 1) { ii = (int)(t / nj); jj = (int)(t % nj); }
    else { jj = (int)(t / ni); ii = (int)(t % ni); }
    int i = ii + oi, j = jj + oj;
    double dm2 = sb(q[I2(qs.s, i - 1, j)], q[I2(qs.s, i - 2, j)]);
    double dm1 = sb(q[I2(qs.s, i, j)], q[I2(qs.s, i - 1, j)]);
    double dp1 = sb(q[I2(qs.s, i + 1, j)], q[I2(qs.s, i, j)]);
    double dp2 = sb(q[I2(qs.s, i + 2, j)], q[I2(qs.s, i + 1, j)]);
    double w = wind[I2(ws.s, ii, jj)];
    long o = I2(os.s, ii, jj);
    out[o] = ad(out[o], ml(w, weno_point(dm2, dm1, dp1, dp2, w, inv_2h, eps)));
}

__global__ void k_weno3(double* out, S3 os, const double* q, S3 qs, const double* wind, S3 ws,
                        int ni, int nj, int nk, int oi, int oj, int ok, double inv_2h,
                        double eps, int p0, int p1, int p2) {
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (t >= (long)ni * nj * nk) return;
    // view axes in order slowest (p0) .. fastest (p2)
    const int d[3] = {ni, nj, nk};
    int idx[3];
    idx[p2] = (int)(t % d[p2]);
    long r = t / d[p2];
    idx[p1] = (int)(r % d[p1]);
    idx[p0] = (int)(r / d[p1]);
    const int ii = idx[0], jj = idx[1], kk = idx[2];
    int i = ii + oi, j = jj + oj, k = kk + ok;
    double dm2 = sb(q[I3(qs.s, i - 1, j, k)], q[I3(qs.s, i - 2, j, k)]);
    double dm1 = sb(q[I3(qs.s, i, j, k)], q[I3(qs.s, i - 1, j, k)]);
    double dp1 = sb(q[I3(qs.s, i + 1, j, k)], q[I3(qs.s, i, j, k)]);
    double dp2 = sb(q[I3(qs.s, i + 2, j, k)], q[I3(qs.s, i + 1, j, k)]);
    double w = wind[I3(ws.s, ii, jj, kk)];
    long o = I3(os.s, ii, jj, kk);
    out[o] = ad(out[o], ml(w, weno_point(dm2, dm1, dp1, dp2, w, inv_2h, eps)));
}

// --------------------------------------------------------------- ghost fill
// PKG/boundary.py:90-156, evaluated point-wise through ghost_value().
struct FillGeo {
    int dim, halo;
    AxisGeo ax[3];
    int ext[3];     // data extents
    long st[3];     // data strides
    long slab_n[3]; // points per slab
    int lo[3][3];   // per slab a, per axis b: first data index
    int cnt[3][3];  // per slab a, per axis b: count
    int olo[3];     // per axis: owned data indices 0..olo-1 on the low side
    int fhi[3];     // per axis: first owned data index on the high side
};

struct DataReader {
    const double* core;
    long st[3];
    __device__ double operator()(int x0, int x1, int x2) const {
        return core[(long)x0 * st[0] + (long)x1 * st[1] + (long)x2 * st[2]];
    }
};

template <int DIM>
__global__ void k_fill(double* data, FillGeo g, BcSpec bc) {
    int a = blockIdx.y;
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (a >= DIM || t >= g.slab_n[a]) return;
    int d[3] = {0, 0, 0};
    long r = t;
    for (int b = DIM - 1; b >= 0; --b) {
        int c = g.cnt[a][b];
        d[b] = g.lo[a][b] + (int)(r % c);
        r /= c;
    }
    // slab a enumerates the two owned ranges of axis a: cnt counts both
    // sides; map the linear index to the lo or hi side
    {
        const int q = d[a] - g.lo[a][a];
        d[a] = q < g.olo[a] ? q : g.fhi[a] + (q - g.olo[a]);
    }
    // core index = data index - (halo - 1)
    int x[3] = {0, 0, 0};
    for (int b = 0; b < DIM; ++b) x[b] = d[b] - (g.halo - 1);
    DataReader rd;
    rd.core = data + (long)(g.halo - 1) * (g.st[0] + g.st[1] + (DIM == 3 ? g.st[2] : 0));
    rd.st[0] = g.st[0];
    rd.st[1] = g.st[1];
    rd.st[2] = DIM == 3 ? g.st[2] : 0;
    double v = ghost_value<DIM>(g.ax, bc, x[0], x[1], DIM == 3 ? x[2] : 0, rd);
    long off = 0;
    for (int b = 0; b < DIM; ++b) off += (long)d[b] * g.st[b];
    data[off] = v;
}

// ------------------------------------------------ numpy-ordered reductions
// numpy pairwise_sum (PW_BLOCKSIZE 128); see oracle/fasmg_oracle.c.
__device__ double pw_leaf(const double* a, long n) {
    if (n < 8) {
        double res = 0.;
        for (long i = 0; i < n; ++i) res = ad(res, a[i]);
        return res;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    long i;
    for (i = 8; i < n - (n % 8); i += 8)
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = ad(r[j], a[i + j]);
    double res = ad(ad(ad(r[0], r[1]), ad(r[2], r[3])), ad(ad(r[4], r[5]), ad(r[6], r[7])));
    for (; i < n; ++i) res = ad(res, a[i]);
    return res;
}

// iterative pairwise recursion over a contiguous buffer (post-order walk of
// numpy's split tree: n2 = n/2 rounded down to a multiple of 8)
__device__ double pw_sum(const double* a, long n) {
    struct Fr { long off, len; int stage; double left; };
    Fr stk[24];
    int sp = 0;
    stk[0].off = 0; stk[0].len = n; stk[0].stage = 0; stk[0].left = 0.0;
    double ret = 0.0;
    while (true) {
        Fr& f = stk[sp];
        if (f.len <= 128) {
            ret = pw_leaf(a + f.off, f.len);
            if (sp == 0) return ret;
            --sp;
            continue;
        }
        long n2 = f.len / 2;
        n2 -= n2 % 8;
        if (f.stage == 0) {
            f.stage = 1;
            ++sp;
            stk[sp].off = f.off; stk[sp].len = n2; stk[sp].stage = 0;
            continue;
        }
        if (f.stage == 1) {
            f.left = ret;
            f.stage = 2;
            ++sp;
            stk[sp].off = f.off + n2; stk[sp].len = f.len - n2; stk[sp].stage = 0;
            continue;
        }
        ret = ad(f.left, ret);
        if (sp == 0) return ret;
        --sp;
    }
}

// Per-chunk gather + pairwise sum of a C-order interior view (numpy buffered
// reduce chunking, oracle or_reduce_chunk).  One thread per chunk; the
// chunk is gathered into a per-thread slice of a scratch buffer.
__global__ void k_chunk_sums(const double* v, S3 vs, int dim, int e0, int e1, int e2,
                             long n, long B, double* scratch, double* sums, long nchunks) {
    long c = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (c >= nchunks) return;
    long start = c * B;
    long len = n - start < B ? n - start : B;
    double* buf = scratch + start;
    for (long t = 0; t < len; ++t) {
        long q = start + t;
        long off;
        if (dim == 2) {
            off = (q / e1) * vs.s[0] + (q % e1) * vs.s[1];
        } else {
            long k = q % e2, r = q / e2;
            off = (r / e1) * vs.s[0] + (r % e1) * vs.s[1] + k * vs.s[2];
        }
        buf[t] = v[off];
    }
    sums[c] = pw_sum(buf, len);
}

// Same per-chunk sums for chunks of exactly 128*2^k (k <= 6) elements --
// the common case (B = 8192 whenever the trailing extents divide 8192):
// numpy's split tree is then a perfect binary tree of 128-element leaves,
// so one CTA gathers the chunk into shared memory (coalesced), 2^k threads
// evaluate the leaves (pw_leaf) and a fixed pairwise tree combines them in
// the recursion's order -- bitwise equal to pw_sum.
constexpr int CH_LEAF = 128, CH_PAD = 129, CH_MAXLEAVES = 64;
__global__ void __launch_bounds__(256) k_chunk_sums_tree(const double* v, S3 vs, int dim, int e0,
                                                         int e1, int e2, long B, int nleaves,
                                                         double* sums) {
    extern __shared__ double sh[];  // [nleaves][CH_PAD] + [nleaves]
    const long c = blockIdx.x;
    const long start = c * B;
    // C-order position (i0, i1, i2) of element start + t, advanced by the
    // CTA width per iteration without 64-bit division
    const int ne = dim == 3 ? e2 : e1;                       // innermost extent
    long q = start + threadIdx.x;
    long row = q / ne;
    int col = (int)(q - row * ne);
    long i0 = dim == 3 ? row / e1 : row;
    int i1 = dim == 3 ? (int)(row - i0 * e1) : col;
    const int step = blockDim.x;
    for (long t = threadIdx.x; t < B; t += step) {
        const long off = dim == 3 ? i0 * vs.s[0] + (long)i1 * vs.s[1] + (long)col * vs.s[2]
                                  : i0 * vs.s[0] + (long)col * vs.s[1];
        sh[(t / CH_LEAF) * CH_PAD + (t % CH_LEAF)] = v[off];
        col += step;
        while (col >= ne) {
            col -= ne;
            if (dim == 3) {
                if (++i1 == e1) { i1 = 0; ++i0; }
            } else {
                ++i0;
            }
        }
    }
    __syncthreads();
    double* leaf = sh + (long)nleaves * CH_PAD;
    if ((int)threadIdx.x < nleaves) leaf[threadIdx.x] = pw_leaf(sh + threadIdx.x * CH_PAD, CH_LEAF);
    __syncthreads();
    for (int w = 1; w < nleaves; w <<= 1) {
        const int i = threadIdx.x * 2 * w;
        if (i + w < nleaves) leaf[i] = ad(leaf[i], leaf[i + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) sums[c] = leaf[0];
}

// The same per-chunk sums when every 128-element leaf lies inside one row of
// the view (innermost extent a multiple of 128 -- every power-of-two grid):
// 8 threads per leaf, thread j summing elements j, j+8, ..., j+120 straight
// from global memory in pw_leaf's accumulator order, the 8 accumulators
// combined by xor-shuffles in pw_leaf's ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
// order, then the chunk's leaf tree as in k_chunk_sums_tree -- bitwise, with
// no shared-memory staging of the chunk.
__global__ void __launch_bounds__(512) k_chunk_sums_leaf(const double* v, S3 vs, int dim, int e1,
                                                         int e2, long B, int nleaves,
                                                         double* sums) {
    __shared__ double leaf[CH_MAXLEAVES];
    const long c = blockIdx.x;
    const int lf = threadIdx.x >> 3, j = threadIdx.x & 7;
    const int ne = dim == 3 ? e2 : e1;
    const long q0 = c * B + (long)lf * CH_LEAF;
    const long row = q0 / ne;
    const long col = q0 - row * ne;
    const long base = dim == 3 ? (row / e1) * vs.s[0] + (row % e1) * vs.s[1] + col * vs.s[2]
                               : row * vs.s[0] + col * vs.s[1];
    const long st = dim == 3 ? vs.s[2] : vs.s[1];
    double x[CH_LEAF / 8];
#pragma unroll
    for (int i = 0; i < CH_LEAF / 8; ++i) x[i] = v[base + (long)(8 * i + j) * st];
    double r = x[0];
#pragma unroll
    for (int i = 1; i < CH_LEAF / 8; ++i) r = ad(r, x[i]);
    const unsigned m = blockDim.x >= 32 ? 0xffffffffu : (1u << blockDim.x) - 1u;
    r = ad(r, __shfl_xor_sync(m, r, 1));
    r = ad(r, __shfl_xor_sync(m, r, 2));
    r = ad(r, __shfl_xor_sync(m, r, 4));
    if (j == 0) leaf[lf] = r;
    __syncthreads();
    for (int w = 1; w < nleaves; w <<= 1) {
        const int i = threadIdx.x * 2 * w;
        if (i + w < nleaves) leaf[i] = ad(leaf[i], leaf[i + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) sums[c] = leaf[0];
}

// np.sum(vals * vals) of an interior view (PKG/grid.py:249): numpy squares
// into a contiguous temporary and runs ONE flat pairwise sum over it.  The
// split tree (n2 = n/2 rounded down to a multiple of 8, leaves <= 128) is
// evaluated level by level, deepest first: node t of depth d is found by
// descending from the root along the bits of t, a leaf squares and sums its
// elements in numpy's 8-accumulator order, an inner node adds its two
// children from the level below.  Level d lives at scratch[2^d - 1 + t].
__device__ __forceinline__ double view_sq(const double* v, S3 vs, int dim, int e1, int e2,
                                          long q) {
    long off;
    if (dim == 2) {
        off = (q / e1) * vs.s[0] + (q % e1) * vs.s[1];
    } else {
        long k = q % e2, r = q / e2;
        off = (r / e1) * vs.s[0] + (r % e1) * vs.s[1] + k * vs.s[2];
    }
    const double x = v[off];
    return ml(x, x);
}

__global__ void k_pw_sumsq_level(const double* v, S3 vs, int dim, int e1, int e2, long n, int d,
                                 double* scratch) {
    const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (t >= (1L << d)) return;
    long off = 0, len = n;
    for (int b = d - 1; b >= 0; --b) {
        if (len <= 128) return;  // a leaf above this depth: no node here
        long n2 = len / 2;
        n2 -= n2 % 8;
        if ((t >> b) & 1) { off += n2; len -= n2; } else { len = n2; }
    }
    double res;
    if (len > 128) {
        const double* lo = scratch + (1L << (d + 1)) - 1;
        res = ad(lo[2 * t], lo[2 * t + 1]);
    } else if (len < 8) {
        res = 0.;
        for (long i = 0; i < len; ++i) res = ad(res, view_sq(v, vs, dim, e1, e2, off + i));
    } else {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = view_sq(v, vs, dim, e1, e2, off + j);
        long i;
        for (i = 8; i < len - (len % 8); i += 8)
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = ad(r[j], view_sq(v, vs, dim, e1, e2, off + i + j));
        res = ad(ad(ad(r[0], r[1]), ad(r[2], r[3])), ad(ad(r[4], r[5]), ad(r[6], r[7])));
        for (; i < len; ++i) res = ad(res, view_sq(v, vs, dim, e1, e2, off + i));
    }
    scratch[(1L << d) - 1 + t] = res;
}

// (the whole CTA stages batches of sums in shared memory with coalesced
// loads; thread 0 adds them in chunk order -- the adds are inherently
// serial, the loads no longer are)
constexpr int CT_BATCH = 4096;
__global__ void __launch_bounds__(1024) k_chunk_total(const double* sums, long nchunks,
                                                      double* out) {
    __shared__ double sh[CT_BATCH];
    double acc = 0.0;
    for (long c0 = 0; c0 < nchunks; c0 += CT_BATCH) {
        const int nb = (int)min((long)CT_BATCH, nchunks - c0);
        for (int j = threadIdx.x; j < nb; j += blockDim.x) sh[j] = sums[c0 + j];
        __syncthreads();
        if (threadIdx.x == 0) {
            int j = 0;
            for (; j + 8 <= nb; j += 8) {
#pragma unroll
                for (int u = 0; u < 8; ++u) acc = ad(acc, sh[j + u]);
            }
            for (; j < nb; ++j) acc = ad(acc, sh[j]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = acc;
}

// interior -= scalar (device scalar: out[0] / count)
__global__ void k_sub_mean(double* v, S3 vs, int dim, int e0, int e1, int e2,
                           const double* total, double count) {
    const double m = dv(total[0], count);
    for (int z = 0; z < box_zn(dim); ++z) {
        int x[3];
        if (!box_coords(dim, e0, e1, e2, z, x)) return;
        const long off = I3(vs.s, x[0], x[1], x[2]);
        v[off] = sb(v[off], m);
    }
}


// ------------------------------------------------------ staggered operators
// gradient_axis (PKG/stencil.py:114-125): out (contiguous, edge-interior
// shape) = (p[x + e_axis] - p[x]) * inv_h
__global__ void k_grad(const double* p, S3 ps, double* out, int dim, int axis, int m0, int m1,
                       int m2, double inv_h) {
    long n = (long)m0 * m1 * (dim == 3 ? m2 : 1);
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (t >= n) return;
    int x[3];
    if (dim == 3) {
        x[2] = 1 + (int)(t % m2);
        long r = t / m2;
        x[1] = 1 + (int)(r % m1);
        x[0] = 1 + (int)(r / m1);
    } else {
        x[1] = 1 + (int)(t % m1);
        x[0] = 1 + (int)(t / m1);
        x[2] = 0;
    }
    long lo = I3(ps.s, x[0], x[1], x[2]);
    long hi = lo + ps.s[axis];
    out[t] = ml(sb(p[hi], p[lo]), inv_h);
}

// divergence_edges_to_cc (PKG/stencil.py:128-156): out interior view =
// sum_axis (c_a[x] - c_a[x - e_a]) * inv_h, accumulated in axis order.
struct Comps { const double* c[3]; S3 s[3]; };
__global__ void k_div(Comps C, double* out, S3 os, int dim, int n0, int n1, int n2,
                      double inv_h) {
    for (int z = 0; z < box_zn(dim); ++z) {
        int x[3];
        if (!box_coords(dim, n0, n1, n2, z, x)) return;  // 0-based interior box position
        const int y0 = x[0] + 1, y1 = x[1] + 1, y2 = dim == 3 ? x[2] + 1 : 0;
        double acc = 0.0;
        for (int a = 0; a < dim; ++a) {
            long hi = I3(C.s[a].s, y0, y1, y2);
            long lo = hi - C.s[a].s[a];
            double term = ml(sb(C.c[a][hi], C.c[a][lo]), inv_h);
            acc = a == 0 ? term : ad(acc, term);
        }
        out[I3(os.s, x[0], x[1], dim == 3 ? x[2] : 0)] = acc;
    }
}

// ------------------------------------------------ projection-step elementwise
// Interior-shaped elementwise ops of the NS drivers (ns.py).  The reference
// has no NS driver; the association order of
// each op is fixed here and mirrored by the oracle composition
// (oracle/ns_oracle.py).
enum NsOp : int {
    NS_MIX_EXT = 0,  // (3a - b) * 0.5         (3u^n - u^{n-1})/2
    NS_MIX_AVG = 1,  // (a + b) * 0.5          (u^n + u~)/2
    NS_AVG4 = 2,     // 0.25 * ((a + b) + (c + d))   PKG/weno.py:51
    NS_AXPY = 3,     // a - s0 * b             u = u~ - dt * grad p~
    NS_ADD = 4,      // a + b                  p = p^n + p~
    NS_COPY = 5,     // a
    NS_RHS1 = 6,     // (a - s0*b) - s0*c      u^n - dt*conv - dt*grad p^n
    NS_RHS2 = 7,     // ((a - s0*b) - s0*c) + s1*d    ... + dt/(2Re) Lap u^n
    NS_NEG = 8,      // -a                     -div u~
};

struct V4 { const double* p[4]; S3 s[4]; };

__global__ void k_ns_elem(int op, double* out, S3 os, V4 in, double s0, double s1, int dim,
                          int e0, int e1, int e2) {
    for (int z = 0; z < box_zn(dim); ++z) {
    int x[3];
    if (!box_coords(dim, e0, e1, e2, z, x)) return;
    double v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
        v[k] = in.p[k] ? in.p[k][I3(in.s[k].s, x[0], x[1], x[2])] : 0.0;
    double r;
    switch (op) {
        case NS_MIX_EXT: r = ml(sb(ml(3.0, v[0]), v[1]), 0.5); break;
        case NS_MIX_AVG: r = ml(ad(v[0], v[1]), 0.5); break;
        case NS_AVG4: r = ml(0.25, ad(ad(v[0], v[1]), ad(v[2], v[3]))); break;
        case NS_AXPY: r = sb(v[0], ml(s0, v[1])); break;
        case NS_ADD: r = ad(v[0], v[1]); break;
        case NS_COPY: r = v[0]; break;
        case NS_RHS1: r = sb(sb(v[0], ml(s0, v[1])), ml(s0, v[2])); break;
        case NS_RHS2: r = ad(sb(sb(v[0], ml(s0, v[1])), ml(s0, v[2])), ml(s1, v[3])); break;
        default: r = -v[0]; break;
    }
    out[I3(os.s, x[0], x[1], x[2])] = r;
    }
}

// Momentum source of one velocity component in ONE pass (the order-1 /
// order-2 RHS of Table 3/5 step 1; order 0: the projection correction
// u~ - dt*gp of step 4): gp = (p[x+e_axis] - p[x]) * inv_h
// (k_grad), lap = (nsum - 2d*u) * inv_h2 (k_lap), then NS_RHS1 / NS_RHS2 --
// the same operations in the same order as those three launches, without
// the two interior-sized temporaries (16 B/DOF of traffic and, at 1024^3,
// 17 GB of memory).  x: 1-based core index of the component's interior.
__global__ void k_ns_rhs(int order, double* out, S3 os, const double* u, S3 us,
                         const double* conv, S3 cs, const double* p, S3 ps, int dim, int axis,
                         int m0, int m1, int m2, double s0, double s1, double inv_h,
                         double inv_h2) {
    for (int zz = 0; zz < box_zn(dim); ++zz) {
    int x[3];
    if (!box_coords(dim, m0, m1, m2, zz, x)) return;
    const int z = dim == 3 ? 1 : 0;
    x[0] += 1;
    x[1] += 1;
    x[2] += z;
    const long pl = I3(ps.s, x[0], x[1], x[2]);
    const double gp = ml(sb(p[pl + ps.s[axis]], p[pl]), inv_h);
    const long uo = I3(us.s, x[0], x[1], x[2]);
    const double uc = u[uo];
    double r;
    if (order == 0) {  // projection correction u = u~ - dt*grad p~ (NS_AXPY)
        r = sb(uc, ml(s0, gp));
    } else {
        const double cv = conv[I3(cs.s, x[0] - 1, x[1] - 1, x[2] - z)];
        r = sb(sb(uc, ml(s0, cv)), ml(s0, gp));
    }
    if (order == 2) {
        double ns = ad(ad(ad(u[uo + us.s[0]], u[uo - us.s[0]]), u[uo + us.s[1]]), u[uo - us.s[1]]);
        if (dim == 3) ns = ad(ad(ns, u[uo + us.s[2]]), u[uo - us.s[2]]);
        const double lap = ml(sb(ns, ml(dim == 3 ? 6.0 : 4.0, uc)), inv_h2);
        r = ad(r, ml(s1, lap));
    }
    out[I3(os.s, x[0] - 1, x[1] - 1, x[2] - z)] = r;
    }
}

// 5/7-point Laplacian (nsum - 2d*c) * inv_h2 (KER/numpy_backend.py:66-88)
__global__ void k_lap(double* out, S3 os, const double* p, S3 ps, int dim, int m0, int m1,
                      int m2, double inv_h2) {
    long n = (long)m0 * m1 * (dim == 3 ? m2 : 1);
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (t >= n) return;
    int x[3];
    if (dim == 3) {
        x[2] = 1 + (int)(t % m2);
        long r = t / m2;
        x[1] = 1 + (int)(r % m1);
        x[0] = 1 + (int)(r / m1);
    } else {
        x[1] = 1 + (int)(t % m1);
        x[0] = 1 + (int)(t / m1);
        x[2] = 0;
    }
    long o = I3(ps.s, x[0], x[1], x[2]);
    double c = p[o];
    double ns = ad(ad(ad(p[o + ps.s[0]], p[o - ps.s[0]]), p[o + ps.s[1]]), p[o - ps.s[1]]);
    if (dim == 3) ns = ad(ad(ns, p[o + ps.s[2]]), p[o - ps.s[2]]);
    out[I3(os.s, x[0] - 1, x[1] - 1, x[2] - (dim == 3 ? 1 : 0))] =
        ml(sb(ns, ml(dim == 3 ? 6.0 : 4.0, c)), inv_h2);
}

}  // namespace fasmg

// ===========================================================================
// C ABI
// ===========================================================================
using namespace fasmg;

static cudaStream_t S(void* s) { return (cudaStream_t)s; }

#define LAUNCH(n, ...)                                                     \
    do {                                                                   \
        if ((n) > 0) __VA_ARGS__;                                          \
        return fasmg_check_launch();                                       \
    } while (0)

extern "C" {

int fasmg_gs_sweep_2d(double* p, const long* ps, const double* f, const long* fs, double b,
                      double h2, double denom, int ilo, int ihi, int jlo, int jhi, int ipar,
                      int jpar, void* stream) {
    int i0 = prng(ilo, ipar), j0 = prng(jlo, jpar);
    if (i0 > ihi || j0 > jhi) return 0;
    int ni = (ihi - i0) / 2 + 1, nj = (jhi - j0) / 2 + 1;
    long n = (long)ni * nj;
    LAUNCH(n, (k_gs2<<<nblk(n, TPB), TPB, 0, S(stream)>>>(p, mk(ps), f, mk(fs), b, h2, denom,
                                                          i0, j0, ni, nj)));
}

int fasmg_gs_sweep_3d(double* p, const long* ps, const double* f, const long* fs, double b,
                      double h2, double denom, int ilo, int ihi, int jlo, int jhi, int klo,
                      int khi, int ipar, int jpar, int kpar, void* stream) {
    int i0 = prng(ilo, ipar), j0 = prng(jlo, jpar), k0 = prng(klo, kpar);
    if (i0 > ihi || j0 > jhi || k0 > khi) return 0;
    int ni = (ihi - i0) / 2 + 1, nj = (jhi - j0) / 2 + 1, nk = (khi - k0) / 2 + 1;
    long n = (long)ni * nj * nk;
    LAUNCH(n, (k_gs3<<<nblk(n, TPB), TPB, 0, S(stream)>>>(p, mk(ps), f, mk(fs), b, h2, denom,
                                                          i0, j0, k0, ni, nj, nk)));
}

int fasmg_apply_op_2d(double* out, const long* os, const double* p, const long* ps, double a,
                      double b, double inv_h2, int ilo, int ihi, int jlo, int jhi,
                      void* stream) {
    int ni = ihi - ilo + 1, nj = jhi - jlo + 1;
    if (ni <= 0 || nj <= 0) return 0;
    long n = (long)ni * nj;
    LAUNCH(n, (k_op2<false><<<nblk(n, TPB), TPB, 0, S(stream)>>>(
                  out, mk(os), p, mk(ps), nullptr, mk(ps), a, b, inv_h2, ilo, jlo, ni, nj)));
}

int fasmg_apply_op_3d(double* out, const long* os, const double* p, const long* ps, double a,
                      double b, double inv_h2, int ilo, int ihi, int jlo, int jhi, int klo,
                      int khi, void* stream) {
    int ni = ihi - ilo + 1, nj = jhi - jlo + 1, nk = khi - klo + 1;
    if (ni <= 0 || nj <= 0 || nk <= 0) return 0;
    long n = (long)ni * nj * nk;
    LAUNCH(n, (k_op3<false><<<nblk(n, TPB), TPB, 0, S(stream)>>>(
                  out, mk(os), p, mk(ps), nullptr, mk(ps), a, b, inv_h2, ilo, jlo, klo, ni,
                  nj, nk)));
}

int fasmg_residual_2d(double* out, const long* os, const double* p, const long* ps,
                      const double* fsrc, const long* fs, double a, double b, double inv_h2,
                      int ilo, int ihi, int jlo, int jhi, void* stream) {
    int ni = ihi - ilo + 1, nj = jhi - jlo + 1;
    if (ni <= 0 || nj <= 0) return 0;
    long n = (long)ni * nj;
    LAUNCH(n, (k_op2<true><<<nblk(n, TPB), TPB, 0, S(stream)>>>(
                  out, mk(os), p, mk(ps), fsrc, mk(fs), a, b, inv_h2, ilo, jlo, ni, nj)));
}

int fasmg_residual_3d(double* out, const long* os, const double* p, const long* ps,
                      const double* fsrc, const long* fs, double a, double b, double inv_h2,
                      int ilo, int ihi, int jlo, int jhi, int klo, int khi, void* stream) {
    int ni = ihi - ilo + 1, nj = jhi - jlo + 1, nk = khi - klo + 1;
    if (ni <= 0 || nj <= 0 || nk <= 0) return 0;
    long n = (long)ni * nj * nk;
    LAUNCH(n, (k_op3<true><<<nblk(n, TPB), TPB, 0, S(stream)>>>(
                  out, mk(os), p, mk(ps), fsrc, mk(fs), a, b, inv_h2, ilo, jlo, klo, ni, nj,
                  nk)));
}

int fasmg_restrict_cc_2d(const double* fine, const long* fs, double* coarse, const long* cs,
                         int m0, int n0, void* stream) {
    long n = (long)m0 * n0;
    LAUNCH(n, (k_rcc2<<<nblk(n, TPB), TPB, 0, S(stream)>>>(fine, mk(fs), coarse, mk(cs), m0,
                                                           n0)));
}

int fasmg_restrict_cc_3d(const double* fine, const long* fs, double* coarse, const long* cs,
                         int m0, int n0, int l0, void* stream) {
    long n = (long)m0 * n0 * l0;
    LAUNCH(n, (k_rcc3<<<nblk(n, TPB), TPB, 0, S(stream)>>>(fine, mk(fs), coarse, mk(cs), m0,
                                                           n0, l0)));
}

int fasmg_prolong_cc_2d(const double* coarse, const long* cs, double* fine, const long* fs,
                        int m0, int n0, void* stream) {
    long n = (long)m0 * n0;
    LAUNCH(n, (k_pcc2<<<nblk(n, TPB), TPB, 0, S(stream)>>>(coarse, mk(cs), fine, mk(fs), m0,
                                                           n0)));
}

int fasmg_prolong_cc_3d(const double* coarse, const long* cs, double* fine, const long* fs,
                        int m0, int n0, int l0, void* stream) {
    long n = (long)m0 * n0 * l0;
    LAUNCH(n, (k_pcc3<<<nblk(n, TPB), TPB, 0, S(stream)>>>(coarse, mk(cs), fine, mk(fs), m0,
                                                           n0, l0)));
}

int fasmg_restrict_edge0_2d(const double* fine, const long* fs, double* coarse,
                            const long* cs, int m0, int n0, void* stream) {
    long n = (long)(m0 - 1) * n0;
    LAUNCH(n, (k_red2<<<nblk(n, TPB), TPB, 0, S(stream)>>>(fine, mk(fs), coarse, mk(cs), m0,
                                                           n0)));
}

int fasmg_restrict_edge0_3d(const double* fine, const long* fs, double* coarse,
                            const long* cs, int m0, int n0, int l0, void* stream) {
    long n = (long)(m0 - 1) * n0 * l0;
    LAUNCH(n, (k_red3<<<nblk(n, TPB), TPB, 0, S(stream)>>>(fine, mk(fs), coarse, mk(cs), m0,
                                                           n0, l0)));
}

int fasmg_prolong_edge0_2d(const double* coarse, const long* cs, double* fine,
                           const long* fs, int m0, int n0, void* stream) {
    long n1 = (long)(m0 + 1) * n0, n2 = (long)m0 * 2 * n0;
    if (n1 > 0)
        k_ped2_lines<<<nblk(n1, TPB), TPB, 0, S(stream)>>>(coarse, mk(cs), fine, mk(fs), m0,
                                                           n0);
    if (n2 > 0) k_ped2_mid<<<nblk(n2, TPB), TPB, 0, S(stream)>>>(fine, mk(fs), m0, n0);
    return fasmg_check_launch();
}

int fasmg_prolong_edge0_3d(const double* coarse, const long* cs, double* fine,
                           const long* fs, int m0, int n0, int l0, void* stream) {
    long n1 = (long)(m0 + 1) * n0 * l0, n2 = (long)m0 * 4 * n0 * l0;
    if (n1 > 0)
        k_ped3_lines<<<nblk(n1, TPB), TPB, 0, S(stream)>>>(coarse, mk(cs), fine, mk(fs), m0,
                                                           n0, l0);
    if (n2 > 0) k_ped3_mid<<<nblk(n2, TPB), TPB, 0, S(stream)>>>(fine, mk(fs), m0, n0, l0);
    return fasmg_check_launch();
}

int fasmg_weno_deriv0_2d(double* out, const long* os, const double* q, const long* qs,
                         const double* wind, const long* ws, int ni, int nj, int oi, int oj,
                         double inv_2h, double eps, void* stream) {
    long n = (long)ni * nj;
    const int fast = labs(os[0]) < labs(os[1]) ? 0 : 1;
    LAUNCH(n, (k_weno2<<<nblk(n, TPB), TPB, 0, S(stream)>>>(out, mk(os), q, mk(qs), wind,
                                                            mk(ws), ni, nj, oi, oj, inv_2h,
                                                            eps, fast)));
}

int fasmg_weno_deriv0_3d(double* out, const long* os, const double* q, const long* qs,
                         const double* wind, const long* ws, int ni, int nj, int nk, int oi,
                         int oj, int ok, double inv_2h, double eps, void* stream) {
    long n = (long)ni * nj * nk;
    int p[3] = {0, 1, 2};  // sort view axes by output stride, largest first
    for (int a = 0; a < 3; ++a)
        for (int b = a + 1; b < 3; ++b)
            if (labs(os[p[b]]) > labs(os[p[a]])) std::swap(p[a], p[b]);
    LAUNCH(n, (k_weno3<<<nblk(n, TPB), TPB, 0, S(stream)>>>(out, mk(os), q, mk(qs), wind,
                                                            mk(ws), ni, nj, nk, oi, oj, ok,
                                                            inv_2h, eps, p[0], p[1], p[2])));
}

int fasmg_weno_convect(double* out, const long* os, const double* const* vel, const long* vst,
                       int dim, int target, int g, const int* ext, double inv_2h, double eps,
                       void* stream) {
    if (dim != 2 && dim != 3) return fasmg_set_error(FASMG_EINVAL, "dim must be 2 or 3");
    Vel3 V;
    memset(&V, 0, sizeof(V));
    for (int a = 0; a < dim; ++a) {
        V.p[a] = vel[a];
        for (int b = 0; b < 3; ++b) V.s[a][b] = b < dim ? vst[3 * a + b] : 0;
    }
    S3 o = mk(os);
    if (dim == 2) o.s[2] = 0;
    const long n = (long)ext[0] * ext[1] * (dim == 3 ? ext[2] : 1);
    if (target < 0 || target >= dim) return fasmg_set_error(FASMG_EINVAL, "bad target axis");
    const int e2 = dim == 3 ? ext[2] : 1;
    if (!box_fits(dim, ext[0], ext[1])) return fasmg_set_error(FASMG_EINVAL, "extent exceeds the 65535 CUDA grid-dimension limit of this launch");
    const dim3 nb = box_grid(dim, ext[0], ext[1], e2), tb = box_block();
    if (n > 0) {
        if (dim == 2) {
            if (target == 0) k_weno_convect<2, 0><<<nb, tb, 0, S(stream)>>>(out, o, V, g, ext[0], ext[1], e2, inv_2h, eps);
            else k_weno_convect<2, 1><<<nb, tb, 0, S(stream)>>>(out, o, V, g, ext[0], ext[1], e2, inv_2h, eps);
        } else {
            if (target == 0) k_weno_convect<3, 0><<<nb, tb, 0, S(stream)>>>(out, o, V, g, ext[0], ext[1], e2, inv_2h, eps);
            else if (target == 1) k_weno_convect<3, 1><<<nb, tb, 0, S(stream)>>>(out, o, V, g, ext[0], ext[1], e2, inv_2h, eps);
            else k_weno_convect<3, 2><<<nb, tb, 0, S(stream)>>>(out, o, V, g, ext[0], ext[1], e2, inv_2h, eps);
        }
    }
    return fasmg_check_launch();
}

// fill_ghosts on a natural-layout C-contiguous data array (PKG/boundary.py:90).
// iface / ext0 serve the axis-0 slab form: interface sides of axis 0 are not
// ghosts (the rows beyond hold a neighbour's data, exchanged beforehand) and
// the local array has ext0 rows along axis 0.
static int fill_ghosts_impl(double* data, int dim, const int* n, int ea, int halo,
                            const int* kinds, const double* vals, int iface, int ext0,
                            cudaStream_t stream) {
    if (dim != 2 && dim != 3) return fasmg_set_error(FASMG_EINVAL, "dim must be 2 or 3");
    FillGeo g;
    BcSpec bc;
    g.dim = dim;
    g.halo = halo;
    for (int a = 0; a < 3; ++a) {
        for (int s = 0; s < 2; ++s) {
            bc.kind[a][s] = a < dim ? kinds[2 * a + s] : 0;
            bc.val[a][s] = a < dim ? vals[2 * a + s] : 0.0;
        }
        g.ax[a].m = a < dim ? n[a] : 1;
        g.ax[a].edge = (a == ea);
        g.ax[a].iface = a == 0 ? iface : 0;
        g.ext[a] = a < dim ? (a == ea ? n[a] + 1 + 2 * (halo - 1) : n[a] + 2 * halo) : 1;
        // owned data indices: low side 0..olo-1, high side fhi..fhi+ohi-1
        const bool edge = (a == ea);
        int olo = edge ? (bc.kind[a][0] == BC_PERIODIC ? halo - 1 : halo) : halo;
        int ohi = halo;  // edge: wall m + rings; cell: halo rings
        if (a == 0 && (iface & 1)) olo = 0;
        if (a == 0 && (iface & 2)) ohi = 0;
        g.olo[a] = olo;
        g.fhi[a] = edge ? halo - 1 + g.ax[a].m : halo + g.ax[a].m;
        g.cnt[a][a] = olo + ohi;  // refined below with lo
        g.lo[a][a] = ohi;         // scratch: ohi until the slab loop
    }
    if (ext0 > 0) g.ext[0] = ext0;
    if (dim == 2) { g.st[1] = 1; g.st[0] = g.ext[1]; g.st[2] = 0; }
    else { g.st[2] = 1; g.st[1] = g.ext[2]; g.st[0] = (long)g.ext[1] * g.ext[2]; }
    int ohi[3];
    for (int a = 0; a < 3; ++a) ohi[a] = g.lo[a][a];
    // slab a: owned along a; not owned along axes b < a; any along b > a.
    long maxn = 0;
    for (int a = 0; a < dim; ++a) {
        long cnt = 1;
        for (int b = 0; b < dim; ++b) {
            int c, lo;
            if (b == a) { lo = 0; c = g.olo[b] + ohi[b]; }
            else if (b < a) {  // up to the high owned rows, or the array end at an interface
                lo = g.olo[b];
                c = (ohi[b] ? g.fhi[b] : g.ext[b]) - g.olo[b];
            }
            else { lo = 0; c = g.ext[b]; }
            g.lo[a][b] = lo;
            g.cnt[a][b] = c;
            cnt *= c;
        }
        g.slab_n[a] = cnt;
        if (cnt > maxn) maxn = cnt;
    }
    if (maxn == 0) return 0;
    dim3 grid(nblk(maxn, TPB), dim);
    if (dim == 2) k_fill<2><<<grid, TPB, 0, stream>>>(data, g, bc);
    else k_fill<3><<<grid, TPB, 0, stream>>>(data, g, bc);
    return fasmg_check_launch();
}

int fasmg_fill_ghosts(double* data, int dim, const int* n, int ea, int halo, const int* kinds,
                      const double* vals, void* stream) {
    return fill_ghosts_impl(data, dim, n, ea, halo, kinds, vals, 0, 0, S(stream));
}

// Axis-0 slab of a field: data is the rank's local
// C-contiguous array with ext0 rows along axis 0, n[0] the rank's cells (an
// edge field with edge axis 0 holds nodes 1..n[0] of the slab, n[0] being the
// wall only on the last rank).  Sides flagged in iface (bit 0 lo, bit 1 hi)
// are rank interfaces: their rows were filled from the neighbour (interior
// values) and are only completed along axes 1..d-1, which is exactly what
// the whole-field fill produces on those rows (every rule of axes >= 1 reads
// its own row).
int fasmg_fill_ghosts_slab(double* data, int dim, const int* n, int ea, int halo,
                           const int* kinds, const double* vals, int iface, int ext0,
                           void* stream) {
    return fill_ghosts_impl(data, dim, n, ea, halo, kinds, vals, iface, ext0, S(stream));
}

// numpy's buffered-reduce chunk length for a C-order view of extent ext
static long np_chunk(int dim, const int* ext) {
    long B = 8192;
    for (int k = 0; k < dim; ++k) {
        long P = 1;
        for (int a = k; a < dim; ++a) P *= ext[a];
        if (P <= 8192) { B = (8192 / P) * P; break; }
    }
    return B;
}

// Per-chunk sums of an interior view, the chunk length B taken from the
// extent gext of the WHOLE array the view belongs to (an axis-0 slab of it:
// the slab must hold whole chunks, so its sums are a contiguous run of the
// global chunk list).  scratch: >= n doubles; sums: >= ceil(n/B) doubles.
int fasmg_view_chunk_sums(const double* v, const long* vs, int dim, const int* ext,
                          const int* gext, double* scratch, double* sums, void* stream) {
    long n = 1;
    for (int a = 0; a < dim; ++a) n *= ext[a];
    const long B = np_chunk(dim, gext);
    bool same = true;
    for (int a = 0; a < dim; ++a) same = same && ext[a] == gext[a];
    if (!same && n % B)
        return fasmg_set_error(FASMG_EINVAL, "slab does not hold whole summation chunks");
    long nch = (n + B - 1) / B;
    S3 s = mk(vs);
    if (dim == 2) s.s[2] = 0;
    int nleaves = 0;  // B = 128 * 2^k, k <= 6, and no partial last chunk
    if (n % B == 0 && B % CH_LEAF == 0) {
        long l = B / CH_LEAF;
        if (l <= CH_MAXLEAVES && (l & (l - 1)) == 0) nleaves = (int)l;
    }
    const int ne = dim == 3 ? ext[2] : ext[1];
    if (nch > 0 && nleaves > 0 && ne % CH_LEAF == 0) {
        k_chunk_sums_leaf<<<(unsigned)nch, 8 * nleaves, 0, S(stream)>>>(
            v, s, dim, ext[1], dim == 3 ? ext[2] : 1, B, nleaves, sums);
    } else if (nch > 0 && nleaves > 0) {
        const size_t shm = sizeof(double) * ((size_t)nleaves * CH_PAD + nleaves);
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_chunk_sums_tree, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(sizeof(double) * (CH_MAXLEAVES * CH_PAD + CH_MAXLEAVES)));
            attr = true;
        }
        k_chunk_sums_tree<<<(unsigned)nch, 256, shm, S(stream)>>>(
            v, s, dim, ext[0], ext[1], dim == 3 ? ext[2] : 1, B, nleaves, sums);
    } else if (nch > 0) {
        k_chunk_sums<<<nblk(nch, 64), 64, 0, S(stream)>>>(v, s, dim, ext[0], ext[1],
                                                          dim == 3 ? ext[2] : 1, n, B, scratch,
                                                          sums, nch);
    }
    return fasmg_check_launch();
}

// Sequential total of nch chunk sums in chunk order into out[0] (device).
int fasmg_chunk_total(const double* sums, long nch, double* out, void* stream) {
    k_chunk_total<<<1, 1024, 0, S(stream)>>>(sums, nch, out);
    return fasmg_check_launch();
}

// np.sum of an interior view in numpy's buffered-reduce order; result into
// out[0] (device).  scratch: >= n doubles; sums: >= ceil(n/B) doubles.
int fasmg_view_sum(const double* v, const long* vs, int dim, const int* ext, double* scratch,
                   double* sums, double* out, void* stream) {
    long n = 1;
    for (int a = 0; a < dim; ++a) n *= ext[a];
    const long nch = (n + np_chunk(dim, ext) - 1) / np_chunk(dim, ext);
    if (int st = fasmg_view_chunk_sums(v, vs, dim, ext, ext, scratch, sums, stream)) return st;
    return fasmg_chunk_total(sums, nch, out, stream);
}

// depth of numpy's pairwise split tree over n elements (its deepest leaf
// lies on the always-right path, whose node sizes are the largest)
static int pw_depth(long n) {
    int d = 0;
    while (n > 128) {
        long n2 = n / 2;
        n2 -= n2 % 8;
        n -= n2;
        ++d;
    }
    return d;
}

// doubles of scratch fasmg_view_sumsq needs for a view of extent ext
long fasmg_view_sumsq_scratch(int dim, const int* ext) {
    long n = 1;
    for (int a = 0; a < dim; ++a) n *= ext[a];
    return (2L << pw_depth(n)) - 1;
}

// out[0] = np.sum(v * v) over a C-order interior view, numpy's flat pairwise
// order (bitwise); scratch holds fasmg_view_sumsq_scratch doubles
int fasmg_view_sumsq(const double* v, const long* vs, int dim, const int* ext, double* scratch,
                     double* out, void* stream) {
    if (dim != 2 && dim != 3) return fasmg_set_error(FASMG_EINVAL, "dim must be 2 or 3");
    long n = 1;
    for (int a = 0; a < dim; ++a) n *= ext[a];
    S3 s = mk(vs);
    if (dim == 2) s.s[2] = 0;
    if (n == 0) return fasmg_check(cudaMemsetAsync(out, 0, sizeof(double), S(stream)));
    const int D = pw_depth(n);
    for (int d = D; d >= 0; --d) {
        const long cnt = 1L << d;
        k_pw_sumsq_level<<<nblk(cnt, 128), 128, 0, S(stream)>>>(v, s, dim, ext[1],
                                                                dim == 3 ? ext[2] : 1, n, d,
                                                                scratch);
        if (int st = fasmg_check_launch()) return st;
    }
    return fasmg_check(cudaMemcpyAsync(out, scratch, sizeof(double), cudaMemcpyDeviceToDevice,
                                       S(stream)));
}

long fasmg_view_sum_chunks(int dim, const int* ext) {
    long n = 1;
    for (int a = 0; a < dim; ++a) n *= ext[a];
    const long B = np_chunk(dim, ext);
    return (n + B - 1) / B;
}

// chunk length numpy uses for a view of extent gext
long fasmg_view_chunk_len(int dim, const int* gext) { return np_chunk(dim, gext); }

// v -= total[0] / count over an interior view (PKG/fas.py:145,156)
int fasmg_sub_mean(double* v, const long* vs, int dim, const int* ext, const double* total,
                   double count, void* stream) {
    long n = (long)ext[0] * ext[1] * (dim == 3 ? ext[2] : 1);
    S3 s = mk(vs);
    if (dim == 2) s.s[2] = 0;
    if (!box_fits(dim, ext[0], ext[1])) return fasmg_set_error(FASMG_EINVAL, "extent exceeds the 65535 CUDA grid-dimension limit of this launch");
    LAUNCH(n, (k_sub_mean<<<box_grid(dim, ext[0], ext[1], dim == 3 ? ext[2] : 1), box_block(), 0,
                            S(stream)>>>(v, s, dim, ext[0], ext[1], dim == 3 ? ext[2] : 1, total,
                                         count)));
}

// gradient_axis: p core view; out contiguous interior of the axis' edge field
int fasmg_gradient_axis(const double* pcore, const long* ps, double* out, int dim,
                        const int* n, int axis, double inv_h, void* stream) {
    int m[3];
    for (int a = 0; a < 3; ++a) m[a] = a < dim ? (a == axis ? n[a] - 1 : n[a]) : 1;
    long tot = (long)m[0] * m[1] * m[2];
    S3 s = mk(ps);
    if (dim == 2) s.s[2] = 0;
    LAUNCH(tot, (k_grad<<<nblk(tot, TPB), TPB, 0, S(stream)>>>(pcore, s, out, dim, axis, m[0],
                                                               m[1], m[2], inv_h)));
}

// divergence: component core views c[a] (strides cs[3a..3a+2]); out is the
// cell interior view (strides os)
int fasmg_divergence(const double* const* comps, const long* cs, double* out, const long* os,
                     int dim, const int* n, double inv_h, void* stream) {
    Comps C;
    for (int a = 0; a < 3; ++a) {
        C.c[a] = a < dim ? comps[a] : nullptr;
        for (int b = 0; b < 3; ++b) C.s[a].s[b] = a < dim ? cs[3 * a + b] : 0;
        if (dim == 2) C.s[a].s[2] = 0;
    }
    S3 o = mk(os);
    if (dim == 2) o.s[2] = 0;
    if (!box_fits(dim, n[0], n[1])) return fasmg_set_error(FASMG_EINVAL, "extent exceeds the 65535 CUDA grid-dimension limit of this launch");
    long tot = (long)n[0] * n[1] * (dim == 3 ? n[2] : 1);
    LAUNCH(tot, (k_div<<<box_grid(dim, n[0], n[1], dim == 3 ? n[2] : 1), box_block(), 0,
                         S(stream)>>>(C, out, o, dim, n[0], n[1], dim == 3 ? n[2] : 1, inv_h)));
}

// generic interior elementwise op (NsOp); views: out + up to 4 inputs
// (NULL allowed), all with element strides [3], extents ext[dim]
int fasmg_ns_elem(int op, double* out, const long* os, const double* const* in,
                  const long* is, double s0, double s1, int dim, const int* ext, void* stream) {
    V4 v;
    for (int k = 0; k < 4; ++k) {
        v.p[k] = in[k];
        for (int b = 0; b < 3; ++b) v.s[k].s[b] = is[3 * k + b];
        if (dim == 2) v.s[k].s[2] = 0;
    }
    S3 o = mk(os);
    if (dim == 2) o.s[2] = 0;
    if (!box_fits(dim, ext[0], ext[1])) return fasmg_set_error(FASMG_EINVAL, "extent exceeds the 65535 CUDA grid-dimension limit of this launch");
    long tot = (long)ext[0] * ext[1] * (dim == 3 ? ext[2] : 1);
    LAUNCH(tot, (k_ns_elem<<<box_grid(dim, ext[0], ext[1], dim == 3 ? ext[2] : 1), box_block(), 0,
                             S(stream)>>>(op, out, o, v, s0, s1, dim, ext[0], ext[1],
                                          dim == 3 ? ext[2] : 1)));
}

// Laplacian of a field at its interior points: p core view, out interior-shaped
// momentum source (k_ns_rhs): out/conv interior views, u and p core views,
// m[dim] the component's interior extents
int fasmg_ns_rhs(int order, double* out, const long* os, const double* ucore, const long* us,
                 const double* conv, const long* cs, const double* pcore, const long* ps,
                 int dim, int axis, const int* m, double s0, double s1, double inv_h,
                 double inv_h2, void* stream) {
    S3 o = mk(os), uu = mk(us), cc = mk(cs), pp = mk(ps);
    if (dim == 2) { o.s[2] = 0; uu.s[2] = 0; cc.s[2] = 0; pp.s[2] = 0; }
    if (!box_fits(dim, m[0], m[1])) return fasmg_set_error(FASMG_EINVAL, "extent exceeds the 65535 CUDA grid-dimension limit of this launch");
    long tot = (long)m[0] * m[1] * (dim == 3 ? m[2] : 1);
    LAUNCH(tot, (k_ns_rhs<<<box_grid(dim, m[0], m[1], dim == 3 ? m[2] : 1), box_block(), 0,
                            S(stream)>>>(
                     order, out, o, ucore, uu, conv, cc, pcore, pp, dim, axis, m[0], m[1],
                     dim == 3 ? m[2] : 1, s0, s1, inv_h, inv_h2)));
}

int fasmg_laplacian(double* out, const long* os, const double* pcore, const long* ps, int dim,
                    const int* m, double inv_h2, void* stream) {
    S3 o = mk(os), pp = mk(ps);
    if (dim == 2) { o.s[2] = 0; pp.s[2] = 0; }
    long tot = (long)m[0] * m[1] * (dim == 3 ? m[2] : 1);
    LAUNCH(tot, (k_lap<<<nblk(tot, TPB), TPB, 0, S(stream)>>>(out, o, pcore, pp, dim, m[0], m[1],
                                                              dim == 3 ? m[2] : 1, inv_h2)));
}

}  // extern "C"
