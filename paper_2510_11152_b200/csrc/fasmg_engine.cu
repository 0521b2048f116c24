// fasmg_engine.cu -- the B200 FAS V-cycle on the parity-blocked layout.
//
// Layout.  A level with n_a cells per axis is stored as 2^d "class" arrays,
// one per index-parity tuple q = (i&1, j&1[, k&1]).  Grid index x_a maps to
// class bit q_a = x_a & 1 and block b_a = (x_a + 1) >> 1, so block b holds
// the 2^d children (2b-1, 2b) of coarse cell b.  Each class array covers
// blocks 0..B_a+1 (B_a = n_a/2) per axis, the last axis contiguous, padded
// so block 1 of every row starts on a 32-byte boundary.
//
// Why: X-MCGS (PKG/smoothers.py:41-45, 136-153) updates one index-parity
// class per color; the first four colors (odd index sum) never read each
// other, nor do the last four, so one smoothing sweep is two dependent
// half-sweeps.  In this layout a half-sweep
// reads the 2^(d-1) opposite classes plus f of its own classes and writes
// its classes: 12 B/DOF, 24 B/DOF per sweep -- the bandwidth minimum -- with
// 256-byte coalesced warp accesses and no parity branching.  Restriction
// and injection become same-index operations across the 2^d classes.
//
// Ghosts.  The reference refills ghosts before every color
// (PKG/smoothers.py:149).  A 5/7-point stencil reads a ghost only through
// the single axis it crosses, and that ghost mirrors either the point
// itself (Dirichlet 2v - p, Neumann copy), the opposite-parity wrap
// (periodic) or a prescribed wall value.  So each class array keeps its
// ghost pads current: whichever kernel writes a boundary point also writes
// the ghost derived from it (fasmg_stencil.cuh), every stencil load is
// branch-free, and no ghost-fill launches are needed -- bitwise identical.
// Edge-centered transfers, which read corner ghosts, use the full
// fill-order chain (ghost_value in fasmg_common.cuh).
//
// Fusions (FAS V-cycle, PKG/fas.py:96-128):
//  * residual + both cell restrictions + FAS tau source in one pass
//    (tau kernel), the coarse operator L_2h(R p) added by a coarse kernel;
//  * the coarse correction c = p_c - R(p) is formed on the fly from the
//    unchanged fine p, so the reference's pinit copy is never stored;
//  * outer residual + sum of squares fused (no residual array).
// The whole V-cycle plus the residual norm is captured once as a CUDA
// graph and replayed per outer iteration.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <limits.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <vector>

#include "fasmg_common.cuh"
#include "fasmg_internal.h"

namespace fasmg {

static constexpr int OFF = 3;  // element offset so block 1 is 32B-aligned
static constexpr int TPB = 256;

struct Lvl {
    int dim, ea;
    int n[3], B[3], E[3];  // B[0], E[0]: LOCAL block-plane count (slab) + pads
    int off0, G0;          // axis-0 global offset of local block 1 (minus 1), global B0
    long s0, s1, cls;  // strides of block axes 0,1 (last axis stride 1)
    long nblk;         // interior blocks
    double h, h2, inv_h2, denom, a, b;
    double rden;       // RN(1/denom) for dvr (host IEEE division)
};

template <int D>
__device__ __forceinline__ long at(const Lvl& L, int c, int b0, int b1, int b2) {
    if (D == 3) return c * L.cls + b0 * L.s0 + b1 * L.s1 + b2 + OFF;
    return c * L.cls + b0 * L.s0 + b1 + OFF;
}

template <int D>
__host__ __device__ __forceinline__ long L_B1(const Lvl& L) { return L.B[1]; }

template <int D>
__device__ __forceinline__ void decode(const Lvl& L, long t, int* bb) {
    if (D == 3) {
        bb[2] = 1 + (int)(t % L.B[2]);
        long r = t / L.B[2];
        bb[1] = 1 + (int)(r % L.B[1]);
        bb[0] = 1 + (int)(r / L.B[1]);
    } else {
        bb[1] = 1 + (int)(t % L.B[1]);
        bb[0] = 1 + (int)(t / L.B[1]);
        bb[2] = 0;
    }
}

template <int D>
__device__ __forceinline__ int qbit(int c, int axis) { return (c >> (D - 1 - axis)) & 1; }

// is (class c, block bb) an interior point? (edge axis: class-0 block B is
// the high wall; axis 0 compares the GLOBAL block index on a slab)
template <int D>
__device__ __forceinline__ bool interior(const Lvl& L, int c, const int* bb) {
    if (L.ea < 0) return true;
    const int g = L.ea == 0 ? bb[0] + L.off0 : bb[L.ea];
    const int B = L.ea == 0 ? L.G0 : L.B[L.ea];
    return !(qbit<D>(c, L.ea) == 0 && g == B);
}

#include "fasmg_stencil.cuh"
#include "fasmg_wave.cuh"
#include "fasmg_coarse.cuh"

// ------------------------------------------------- edge-centered transfers
// Reader of raw stored values at GLOBAL core (grid) index x in the blocked
// layout (on an axis-0 slab the block index is shifted by the slab offset;
// the positions a transfer reads stay within the slab and its halo planes).
template <int D>
struct BlkReader {
    const double* P;
    Lvl L;
    __device__ double operator()(int x0, int x1, int x2) const {
        int x[3] = {x0, x1, x2};
        int c = 0, b[3] = {0, 0, 0};
#pragma unroll
        for (int a = 0; a < D; ++a) {
            c |= (x[a] & 1) << (D - 1 - a);
            b[a] = (x[a] + 1) >> 1;
        }
        b[0] -= L.off0;
        return P[at<D>(L, c, b[0], b[1], b[2])];
    }
};

template <int D>
__device__ __forceinline__ double gval(const double* P, const Lvl& L, const BcSpec& bc, int x0,
                                       int x1, int x2) {
    AxisGeo ax[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        ax[a].m = a < D ? L.n[a] : 1;
        ax[a].edge = (a == L.ea);
    }
    BlkReader<D> rd{P, L};
    return ghost_value<D>(ax, bc, x0, x1, x2, rd);
}

// Fine value at grid index x with ghosts filled under bc: fast path for
// interior points.
template <int D>
__device__ __forceinline__ double fval(const double* P, const Lvl& L, const BcSpec& bc,
                                       const int* x) {
    bool in = true;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        int hi = (a == L.ea) ? L.n[a] - 1 : L.n[a];
        in = in && x[a] >= 1 && x[a] <= hi;
    }
    if (in) {
        BlkReader<D> rd{P, L};
        return rd(x[0], x[1], D == 3 ? x[2] : 0);
    }
    return gval<D>(P, L, bc, x[0], x[1], D == 3 ? x[2] : 0);
}

// restrict_edge (PKG/transfer.py:76-91; KER/numpy_backend.py:162-191) for
// edge axis ea: the reference runs the axis-0 kernel on a moveaxis view
// whose axes are (ea, remaining axes in order).  Thread per coarse interior
// point; writes coarse value into the blocked coarse array.
template <int D>
__global__ void __launch_bounds__(TPB) k_restrict_edge(const double* __restrict__ Fn, Lvl L,
                                                       BcSpec bc, double* __restrict__ Co,
                                                       Lvl Lc) {
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    // enumerate coarse interior points in natural order
    long m[3];
    const int ea = L.ea;
    for (int a = 0; a < 3; ++a) m[a] = a < D ? (a == ea ? Lc.n[a] - 1 : Lc.n[a]) : 1;
    if (t >= m[0] * m[1] * m[2]) return;
    int I[3];
    I[2] = 1 + (int)(t % m[2]);
    long r = t / m[2];
    I[1] = 1 + (int)(r % m[1]);
    I[0] = 1 + (int)(r / m[1]);
    if (D == 2) { I[2] = 0; I[1] = 1 + (int)(t % m[1]); I[0] = 1 + (int)(t / m[1]); }
    // permuted axes: v0 = ea, v1, v2 = others in order
    int pa[3];
    pa[0] = ea;
    {
        int q = 1;
        for (int a = 0; a < D; ++a)
            if (a != ea) pa[q++] = a;
    }
    int fi = 2 * I[pa[0]], fj = 2 * I[pa[1]], fk = D == 3 ? 2 * I[pa[2]] : 0;
    auto F = [&](int x, int y, int z) {
        int g[3];
        g[pa[0]] = x;
        g[pa[1]] = y;
        if (D == 3) g[pa[2]] = z;
        else g[2] = 0;
        return fval<D>(Fn, L, bc, g);
    };
    double res;
    if (D == 2) {
        double t1 = ad(ad(F(fi - 1, fj - 1, 0), ml(2.0, F(fi - 1, fj, 0))), F(fi - 1, fj + 1, 0));
        double t2 = ad(ad(F(fi, fj - 1, 0), ml(2.0, F(fi, fj, 0))), F(fi, fj + 1, 0));
        res = ml(ad(t1, t2), 0.125);
    } else {
        double tang[2];
#pragma unroll
        for (int cI = 0; cI < 2; ++cI) {
            int fx = fi - 1 + cI;
            double rows[3];
#pragma unroll
            for (int rr = 0; rr < 3; ++rr) {
                int fy = fj - 1 + rr;
                rows[rr] = ml(ad(ad(F(fx, fy, fk - 1), ml(2.0, F(fx, fy, fk))), F(fx, fy, fk + 1)),
                              0.25);
            }
            tang[cI] = ml(ad(ad(rows[0], ml(2.0, rows[1])), rows[2]), 0.25);
        }
        res = ml(ad(tang[0], tang[1]), 0.5);
    }
    int cc = 0, cb[3] = {0, 0, 0};
#pragma unroll
    for (int a = 0; a < D; ++a) {
        cc |= (I[a] & 1) << (D - 1 - a);
        cb[a] = (I[a] + 1) >> 1;
    }
    Co[at<D>(Lc, cc, cb[0], cb[1], cb[2])] = res;
}

// PINIT = P_c (interior) for edge fields
template <int D>
__global__ void k_copy_blk(const double* __restrict__ src, double* __restrict__ dst, long n) {
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (t < n) dst[t] = src[t];
}

// Correction value c = p_c - pinit at coarse grid index x, with homogenized
// ghosts (PKG/fas.py:119-121).  The periodic low wall of p_c is never
// written in the reference (zero for solver-owned coarse fields) and the
// interior subtraction leaves it unchanged.
template <int D>
struct CorrReader {
    const double* Pc;
    const double* PI;
    Lvl L;
    __device__ double operator()(int x0, int x1, int x2) const {
        int x[3] = {x0, x1, x2};
        int c = 0, b[3] = {0, 0, 0};
        bool wall = false;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            c |= (x[a] & 1) << (D - 1 - a);
            b[a] = (x[a] + 1) >> 1;
            if (a == L.ea && x[a] == 0) wall = true;
        }
        b[0] -= L.off0;
        long o = at<D>(L, c, b[0], b[1], b[2]);
        if (wall) return Pc[o];
        return sb(Pc[o], PI[o]);
    }
};

// prolong_edge (PKG/transfer.py:94-109; KER/numpy_backend.py:194-224) of the
// correction, added to the fine interior (PKG/fas.py:122-123).  Thread per
// fine interior point.
template <int D>
__global__ void __launch_bounds__(TPB) k_correct_edge(double* __restrict__ P, Lvl L,
                                                      const double* __restrict__ Pc,
                                                      const double* __restrict__ PI, Lvl Lc,
                                                      BcSpec bch) {
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (t >= L.nblk) return;
    int bb[3];
    decode<D>(L, t, bb);
    const int ea = L.ea;
    int pa[3];
    pa[0] = ea;
    {
        int q = 1;
        for (int a = 0; a < D; ++a)
            if (a != ea) pa[q++] = a;
    }
    AxisGeo ax[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        ax[a].m = a < D ? Lc.n[a] : 1;
        ax[a].edge = (a == ea);
    }
    CorrReader<D> rd{Pc, PI, Lc};
    // coarse value at permuted coarse index (i, j, k)
    auto C = [&](int i, int j, int k) {
        int g[3];
        g[pa[0]] = i;
        g[pa[1]] = j;
        if (D == 3) g[pa[2]] = k;
        else g[2] = 0;
        bool in = true;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            int hi = (a == ea) ? Lc.n[a] - 1 : Lc.n[a];
            in = in && g[a] >= 1 && g[a] <= hi;
        }
        if (in) return rd(g[0], g[1], D == 3 ? g[2] : 0);
        return ghost_value<D>(ax, bch, g[0], g[1], D == 3 ? g[2] : 0, rd);
    };
    // value of the prolonged field on coarse line i (fine column 2i) at fine
    // tangential indices (fy, fz)
    auto line = [&](int i, int fy, int fz) {
        int j = (fy + 1) >> 1, dj = (fy & 1) ? -1 : 1;
        if (D == 2) return ml(ad(ml(3.0, C(i, j, 0)), C(i, j + dj, 0)), 0.25);
        int k = (fz + 1) >> 1, dk = (fz & 1) ? -1 : 1;
        double t_near = ml(ad(ml(3.0, C(i, j, k)), C(i, j + dj, k)), 0.25);
        double t_far = ml(ad(ml(3.0, C(i, j, k + dk)), C(i, j + dj, k + dk)), 0.25);
        return ml(ad(ml(3.0, t_near), t_far), 0.25);
    };
#pragma unroll
    for (int c = 0; c < (1 << D); ++c) {
        if (!interior<D>(L, c, bb)) continue;
        int x[3] = {0, 0, 0};
#pragma unroll
        for (int a = 0; a < D; ++a) x[a] = 2 * bb[a] - qbit<D>(c, a);
        int fx = x[pa[0]], fy = x[pa[1]], fz = D == 3 ? x[pa[2]] : 0;
        double v;
        if ((fx & 1) == 0) v = line(fx >> 1, fy, fz);
        else v = ml(ad(line(fx >> 1, fy, fz), line((fx >> 1) + 1, fy, fz)), 0.5);
        const long o = at<D>(L, c, bb[0], bb[1], bb[2]);
        P[o] = ad(P[o], v);
    }
}

// ---------------------------------------------- fast edge-field transfers
// The transfers above evaluate the reference's ghost chain per read.  The
// fast path first materialises every ghost / corner a transfer reads into
// the blocked array's pad slots (k_pad_all), or the correction c = p_c -
// pinit with its homogenized ghosts into a scratch array (k_corr_edge), and
// then reads raw values: same values, same arithmetic, no per-read chains.

// grid index of (class c, block b) along axis a, and whether a transfer
// may read it (cell axis 0..n+1, edge axis 0..n)
template <int D>
__device__ __forceinline__ bool grid_idx(const Lvl& L, int c, const int* b, int* x, bool* inner) {
    bool in = true;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        x[a] = 2 * (b[a] + (a == 0 ? L.off0 : 0)) - qbit<D>(c, a);  // global index
        const bool edge = a == L.ea;
        const int hi = edge ? L.n[a] : L.n[a] + 1;
        if (x[a] < 0 || x[a] > hi) return false;
        in = in && x[a] >= 1 && x[a] <= (edge ? L.n[a] - 1 : L.n[a]);
    }
    *inner = in;
    return true;
}

// Every pad slot (faces, edges, corners) of a level's blocked array set to
// the value fill_ghosts gives it under bc (PKG/boundary.py:90-156).  Thread
// per pad block position of one face (grid.y = face), all classes.
template <int D>
__device__ __forceinline__ void pad_all_pt(double* __restrict__ P, const Lvl& L,
                                           const BcSpec& bc, int face, int i1, int i2) {
    const int a = face >> 1, side = face & 1;
    int oth[2], no = 0;
#pragma unroll
    for (int q = 0; q < D; ++q)
        if (q != a) oth[no++] = q;
    if (i1 >= L.E[oth[0]] || (D == 3 ? i2 >= L.E[oth[1]] : i2 > 0)) return;
    int b[3] = {0, 0, 0};
    b[a] = side ? L.B[a] + 1 : 0;
    b[oth[0]] = i1;
    if (D == 3) b[oth[1]] = i2;
    AxisGeo ax[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        ax[q].m = q < D ? L.n[q] : 1;
        ax[q].edge = (q == L.ea);
    }
    BlkReader<D> rd{P, L};
    // all classes' ghost values before any store: the chains end in reads
    // of interior points (or the never-written periodic low wall), never in
    // a slot written here, so their loads can all be in flight at once
    double v[1 << D];
    unsigned todo = 0u;
#pragma unroll
    for (int c = 0; c < (1 << D); ++c) {
        int x[3] = {0, 0, 0};
        bool in;
        v[c] = 0.0;
        if (!grid_idx<D>(L, c, b, x, &in) || in) continue;
        todo |= 1u << c;
        v[c] = ghost_value<D>(ax, bc, x[0], x[1], x[2], rd);
    }
#pragma unroll
    for (int c = 0; c < (1 << D); ++c)
        if ((todo >> c) & 1u) P[at<D>(L, c, b[0], b[1], b[2])] = v[c];
}

// grid: x over the face's last other axis (3D; 2D: the other axis), y over
// the first other axis (3D), z = face (+ 2D for the second array of
// k_pad_all2) -- no integer division
template <int D>
__device__ __forceinline__ void pad_face_coords(int& i1, int& i2) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (D == 3) { i1 = blockIdx.y; i2 = i; }
    else { i1 = i; i2 = 0; }
}

template <int D>
__global__ void __launch_bounds__(TPB) k_pad_all(double* __restrict__ P, Lvl L, BcSpec bc) {
    int i1, i2;
    pad_face_coords<D>(i1, i2);
    pad_all_pt<D>(P, L, bc, blockIdx.z, i1, i2);
}

// the pads of two arrays of one level in one launch (P under bc, R under
// bch) -- the edge tau pass pads p and r together
template <int D>
__global__ void __launch_bounds__(TPB) k_pad_all2(double* __restrict__ P, BcSpec bc,
                                                  double* __restrict__ R, BcSpec bch, Lvl L) {
    int i1, i2;
    pad_face_coords<D>(i1, i2);
    const int face = blockIdx.z % (2 * D);
    if (blockIdx.z < 2 * D) pad_all_pt<D>(P, L, bc, face, i1, i2);
    else pad_all_pt<D>(R, L, bch, face, i1, i2);
}

// coarse rows along axis 0 a fine level's blocks restrict to: all m0 of
// them, or on a slab those of the local blocks off0+1..off0+B0 (fine block
// I <-> coarse index I) that are interior
__host__ __device__ __forceinline__ long restrict_rows(const Lvl& L, long m0) {
    const long r = (long)L.B[0] < m0 - L.off0 ? (long)L.B[0] : m0 - L.off0;
    return r > 0 ? r : 0;
}

// restrict_edge on raw reads (pads of Fn filled by k_pad_all).  Thread per
// coarse interior point I (natural order, last axis fastest): fine edge-
// axis columns 2I-1 (class bit 1) and 2I (bit 0) of block I; tangential
// rows 2J-1 (bit 1, block J), 2J (bit 0, block J), 2J+1 (bit 1, block J+1).
// The edge axis is a template parameter so every class/offset is a
// compile-time constant; the arithmetic is KER/numba_backend.py:304-342.
template <int D, int EA>
__device__ __forceinline__ void restrict_edge_pt(const double* __restrict__ Fn, const Lvl& L,
                                                 double* __restrict__ Co, const Lvl& Lc, long t) {
    constexpr int P0 = EA < 0 ? 0 : EA, P1 = P0 == 0 ? 1 : 0, P2 = D == 3 ? (P0 == 2 ? 1 : 2) : 0;
    long m[3];
    for (int a = 0; a < 3; ++a) m[a] = a < D ? (a == P0 ? Lc.n[a] - 1 : Lc.n[a]) : 1;
    // axis 0 on a slab: the coarse points of this rank's fine blocks
    m[0] = restrict_rows(L, m[0]);
    if (t >= m[0] * m[1] * m[2]) return;
    int I[3];
    if (D == 3) {
        I[2] = 1 + (int)(t % m[2]);
        long r = t / m[2];
        I[1] = 1 + (int)(r % m[1]);
        I[0] = 1 + (int)(r / m[1]);
    } else {
        I[2] = 0;
        I[1] = 1 + (int)(t % m[1]);
        I[0] = 1 + (int)(t / m[1]);
    }
    const long base = at<D>(L, 0, I[0], I[1], D == 3 ? I[2] : 0);
    I[0] += L.off0;  // global coarse index from here on
    // fine value: edge offset de (0: 2I-1, 1: 2I), tangential dj/dk (0: 2J-1,
    // 1: 2J, 2: 2J+1)
    auto F = [&](int de, int dj, int dk) {
        int c = 0;
        long o = base;
        c |= (de == 0 ? 1 : 0) << (D - 1 - P0);
        c |= (dj == 1 ? 0 : 1) << (D - 1 - P1);
        if (dj == 2) o += bstride<D>(L, P1);
        if (D == 3) {
            c |= (dk == 1 ? 0 : 1) << (D - 1 - P2);
            if (dk == 2) o += bstride<D>(L, P2);
        }
        return Fn[o + (long)c * L.cls];
    };
    double res;
    if (D == 2) {
        const double t1 = ad(ad(F(0, 0, 0), ml(2.0, F(0, 1, 0))), F(0, 2, 0));
        const double t2 = ad(ad(F(1, 0, 0), ml(2.0, F(1, 1, 0))), F(1, 2, 0));
        res = ml(ad(t1, t2), 0.125);
    } else {
        double tang[2];
#pragma unroll
        for (int cI = 0; cI < 2; ++cI) {
            double rows[3];
#pragma unroll
            for (int rr = 0; rr < 3; ++rr)
                rows[rr] = ml(ad(ad(F(cI, rr, 0), ml(2.0, F(cI, rr, 1))), F(cI, rr, 2)), 0.25);
            tang[cI] = ml(ad(ad(rows[0], ml(2.0, rows[1])), rows[2]), 0.25);
        }
        res = ml(ad(tang[0], tang[1]), 0.5);
    }
    int cc = 0, cb[3] = {0, 0, 0};
#pragma unroll
    for (int a = 0; a < D; ++a) {
        cc |= (I[a] & 1) << (D - 1 - a);
        cb[a] = (I[a] + 1) >> 1;
    }
    cb[0] -= Lc.off0;
    Co[at<D>(Lc, cc, cb[0], cb[1], cb[2])] = res;
}

template <int D, int EA>
__global__ void __launch_bounds__(TPB) k_restrict_edge_fast(const double* __restrict__ Fn, Lvl L,
                                                            double* __restrict__ Co, Lvl Lc) {
    restrict_edge_pt<D, EA>(Fn, L, Co, Lc, blockIdx.x * (long)blockDim.x + threadIdx.x);
}

// Corr = the value CorrReader + ghost chain give at every coarse position a
// prolongation reads (interior: p_c - pinit; ghosts under the homogenized
// bc).  Thread per block position (pads included) of the coarse level, all
// 2^d classes: a 2D/3D thread tile (block axes from the grid, no 64-bit
// div/mod); interior points are one subtraction, only pad positions take
// the ghost chain.
template <int D>
__device__ __forceinline__ void corr_edge_pt(const double* __restrict__ Pc,
                                             const double* __restrict__ PI, const Lvl& Lc,
                                             const BcSpec& bch, double* __restrict__ Corr,
                                             const int* b, bool skip_inner = false) {
    const long o0 = at<D>(Lc, 0, b[0], b[1], b[2]);
    CorrReader<D> rd{Pc, PI, Lc};
    // (skip_inner: the interior points of interior blocks are k_corr_edge_in's)
    bool inner_blk = skip_inner;
#pragma unroll
    for (int a = 0; a < D; ++a) inner_blk = inner_blk && b[a] >= 1 && b[a] <= Lc.B[a];
    // values of every class first, then the stores (the loads in flight
    // together)
    double v[1 << D];
    unsigned todo = 0u;
#pragma unroll
    for (int c = 0; c < (1 << D); ++c) {
        int x[3] = {0, 0, 0};
        bool in;
        v[c] = 0.0;
        if (!grid_idx<D>(Lc, c, b, x, &in)) continue;
        if (inner_blk && in) continue;
        todo |= 1u << c;
        const long o = o0 + (long)c * Lc.cls;
        if (in) {
            v[c] = sb(Pc[o], PI[o]);
        } else {
            AxisGeo ax[3];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                ax[q].m = q < D ? Lc.n[q] : 1;
                ax[q].edge = (q == Lc.ea);
            }
            v[c] = ghost_value<D>(ax, bch, x[0], x[1], x[2], rd);
        }
    }
#pragma unroll
    for (int c = 0; c < (1 << D); ++c)
        if ((todo >> c) & 1u) Corr[o0 + (long)c * Lc.cls] = v[c];
}

// The interior part of Corr (the common case of corr_edge_pt), on the block
// tile of the coarse level's interior blocks: one subtraction per interior
// point, without the ghost chain's registers and stack frame.
template <int D>
__global__ void __launch_bounds__(TPB) k_corr_edge_in(const double* __restrict__ Pc,
                                                      const double* __restrict__ PI, Lvl Lc,
                                                      double* __restrict__ Corr) {
    int bb[3];
    if (!tile_coords<D>(Lc, bb)) return;
    const long o0 = at<D>(Lc, 0, bb[0], bb[1], bb[2]);
#pragma unroll
    for (int c = 0; c < (1 << D); ++c) {
        int x[3] = {0, 0, 0};
        bool in;
        if (!grid_idx<D>(Lc, c, bb, x, &in) || !in) continue;
        const long o = o0 + (long)c * Lc.cls;
        Corr[o] = sb(Pc[o], PI[o]);
    }
}

template <int D>
__global__ void __launch_bounds__(TPB) k_corr_edge(const double* __restrict__ Pc,
                                                   const double* __restrict__ PI, Lvl Lc,
                                                   BcSpec bch, double* __restrict__ Corr,
                                                   int skip_inner = 0) {
    int b[3] = {0, 0, 0};
    if (D == 3) {
        b[2] = blockIdx.x * blockDim.x + threadIdx.x;
        b[1] = blockIdx.y * blockDim.y + threadIdx.y;
        b[0] = blockIdx.z;
        if (b[2] >= Lc.E[2] || b[1] >= Lc.E[1]) return;
    } else {
        b[1] = blockIdx.x * blockDim.x + threadIdx.x;
        b[0] = blockIdx.y * blockDim.y + threadIdx.y;
        if (b[1] >= Lc.E[1] || b[0] >= Lc.E[0]) return;
    }
    corr_edge_pt<D>(Pc, PI, Lc, bch, Corr, b, skip_inner != 0);
}

// The non-interior part of Corr (ghost chain): only the block positions on
// the six faces of the block box (0 or B+1 along an axis) and, for an edge
// field, the high wall plane (block B along the edge axis, whose class-0
// points are the wall) -- grid (x, y) over the other two axes, z = plane.
template <int D>
__global__ void __launch_bounds__(TPB) k_corr_edge_pads(const double* __restrict__ Pc,
                                                        const double* __restrict__ PI, Lvl Lc,
                                                        BcSpec bch, double* __restrict__ Corr) {
    const int z = blockIdx.z;
    int a, pos;
    if (z < 2 * D) {
        a = z >> 1;
        pos = (z & 1) ? Lc.B[a] + 1 : 0;
    } else {
        a = Lc.ea;  // the wall plane (launched for edge fields only)
        pos = Lc.B[a];
    }
    int oth[2] = {0, 0}, no = 0;
    for (int t = 0; t < D; ++t)
        if (t != a) oth[no++] = t;
    int b[3] = {0, 0, 0};
    b[a] = pos;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (D == 3) {
        b[oth[0]] = blockIdx.y;
        b[oth[1]] = i;
        if (b[oth[0]] >= Lc.E[oth[0]] || b[oth[1]] >= Lc.E[oth[1]]) return;
    } else {
        b[oth[0]] = i;
        if (blockIdx.y || b[oth[0]] >= Lc.E[oth[0]]) return;
    }
    corr_edge_pt<D>(Pc, PI, Lc, bch, Corr, b, true);
}

// launch geometry of k_corr_edge: every block position 0..E-1 per axis
template <int D>
static void corr_edge_grid(const Lvl& Lc, dim3& grd, dim3& blk) {
    blk = dim3(32, 8, 1);
    if (D == 3) grd = dim3((Lc.E[2] + 31) / 32, (Lc.E[1] + 7) / 8, Lc.E[0]);
    else grd = dim3((Lc.E[1] + 31) / 32, (Lc.E[0] + 7) / 8, 1);
}

// prolong_edge of Corr added to the fine interior (raw reads).  All 2^d
// fine points of block bb draw on the same 2 x 3 (x 3) coarse neighbourhood
// (edge-axis lines b-1, b; tangential b-1..b+1), loaded once into
// registers; with the edge axis a template parameter every index below is
// a compile-time constant.  Per fine point with parity bits (qe, qj, qk) in
// the permuted axes (edge axis first): tangential j = b, j+dj = b-1 (q=1)
// or b+1 (q=0); edge-axis line b (qe=0) or the mean of lines b-1, b (qe=1)
// -- KER/numpy_backend.py:194-224.
template <int D, int EA>
__device__ __forceinline__ void correct_edge_pt(double* __restrict__ P, const Lvl& L,
                                                const double* __restrict__ Corr, const Lvl& Lc,
                                                const int* bb) {
    constexpr int P0 = EA < 0 ? 0 : EA, P1 = P0 == 0 ? 1 : 0, P2 = D == 3 ? (P0 == 2 ? 1 : 2) : 0;
    const int gb[3] = {bb[0] + L.off0, bb[1], bb[2]};  // global block (axis-0 slab)
    const int be = gb[P0], bj = gb[P1], bk = D == 3 ? gb[P2] : 0;
    // the block's fine values first (independent of the coarse loads below)
    const long o0 = at<D>(L, 0, bb[0], bb[1], bb[2]);
    double pv[1 << D];
#pragma unroll
    for (int c = 0; c < (1 << D); ++c) pv[c] = P[o0 + (long)c * L.cls];
    BlkReader<D> rd{Corr, Lc};
    double cv[2][3][3];
#pragma unroll
    for (int di = 0; di < 2; ++di)
#pragma unroll
        for (int dj = 0; dj < 3; ++dj)
#pragma unroll
            for (int dk = 0; dk < 3; ++dk) {
                if (D == 2 && dk > 0) { cv[di][dj][dk] = 0.0; continue; }
                int g[3] = {0, 0, 0};
                g[P0] = be - 1 + di;
                g[P1] = bj - 1 + dj;
                if (D == 3) g[P2] = bk - 1 + dk;
                cv[di][dj][dk] = rd(g[0], g[1], g[2]);
            }
#pragma unroll
    for (int c = 0; c < (1 << D); ++c) {
        if (!interior<D>(L, c, bb)) continue;
        const int qe = qbit<D>(c, P0), qj = qbit<D>(c, P1), qk = D == 3 ? qbit<D>(c, P2) : 0;
        const int jd = qj ? 0 : 2, kd = qk ? 0 : 2;
        auto line = [&](int i) {
            if (D == 2) return ml(ad(ml(3.0, cv[i][1][0]), cv[i][jd][0]), 0.25);
            const double t_near = ml(ad(ml(3.0, cv[i][1][1]), cv[i][jd][1]), 0.25);
            const double t_far = ml(ad(ml(3.0, cv[i][1][kd]), cv[i][jd][kd]), 0.25);
            return ml(ad(ml(3.0, t_near), t_far), 0.25);
        };
        const double v = qe ? ml(ad(line(0), line(1)), 0.5) : line(1);
        P[o0 + (long)c * L.cls] = ad(pv[c], v);
    }
}

template <int D, int EA>
__global__ void __launch_bounds__(TPB, 4) k_correct_edge_fast(double* __restrict__ P, Lvl L,
                                                           const double* __restrict__ Corr,
                                                           Lvl Lc) {
    int bb[3];
    if (!tile_coords<D>(L, bb)) return;  // 2D/3D thread tile: no 64-bit div/mod
    correct_edge_pt<D, EA>(P, L, Corr, Lc, bb);
}

__global__ void k_final_sum(const double* __restrict__ part, int n, double* out) {
    __shared__ double sh[1024];
    double acc = 0.0;
    // the same order as one load per iteration, with 8 loads in flight
    const int step = blockDim.x;
    int i = threadIdx.x;
    for (; i + 7 * step < n; i += 8 * step) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = part[i + u * step];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = ad(acc, x[u]);
    }
    for (; i < n; i += step) acc = ad(acc, part[i]);
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) sh[threadIdx.x] = ad(sh[threadIdx.x], sh[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = sh[0];
}

// ------------------------------------------------------- pack / unpack
// natural core view (strides) <-> blocked arrays.  pack covers core
// indices 0..M+1 (cell) / 0..n (edge axis) so stored walls travel too.
template <int D>
__global__ void k_pack(const double* __restrict__ src, long s0, long s1, long s2,
                       double* __restrict__ dst, Lvl L, int e0, int e1, int e2) {
    // 2D/3D thread tile, no 64-bit div/mod.  A thread moves the pair
    // (2j, 2j+1) of the contiguous axis: class bit 0 of block j and class
    // bit 1 of block j+1, so a warp reads 64 consecutive doubles and writes
    // 32 consecutive doubles into each of two class arrays.
    constexpr int LA = D - 1;  // contiguous axis
    int x[3] = {0, 0, 0};
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (D == 3) {
        x[1] = blockIdx.y * blockDim.y + threadIdx.y;
        x[0] = blockIdx.z;
        if (2 * j >= e2 || x[1] >= e1) return;
    } else {
        x[0] = blockIdx.y * blockDim.y + threadIdx.y;
        if (2 * j >= e1 || x[0] >= e0) return;
    }
    const int eL = D == 3 ? e2 : e1;
    const long sL = D == 3 ? s2 : s1;
    const long so = (long)x[0] * s0 + (D == 3 ? (long)x[1] * s1 : 0) + (long)(2 * j) * sL;
    const bool two = 2 * j + 1 < eL;
    const double v0 = src[so];
    const double v1 = two ? src[so + sL] : 0.0;
    int c = 0, b[3] = {0, 0, 0};
#pragma unroll
    for (int a = 0; a < LA; ++a) {
        c |= (x[a] & 1) << (D - 1 - a);
        b[a] = (x[a] + 1) >> 1;
    }
    b[LA] = j;  // x = 2j: class bit 0, block j
    dst[at<D>(L, c, b[0], b[1], b[2])] = v0;
    if (two) {  // x = 2j + 1: class bit 1, block j + 1
        b[LA] = j + 1;
        dst[at<D>(L, c | 1, b[0], b[1], b[2])] = v1;
    }
}

// interior only (core indices 1..M).  A thread moves the pair (2j-1, 2j) of
// the contiguous axis: classes bit 1 and bit 0 of block j.
template <int D>
__global__ void k_unpack(const double* __restrict__ src, Lvl L, double* __restrict__ dst,
                         long s0, long s1, long s2, int m0, int m1, int m2) {
    constexpr int LA = D - 1;
    int x[3] = {0, 0, 0};
    const int j = 1 + (int)(blockIdx.x * blockDim.x + threadIdx.x);
    if (D == 3) {
        x[1] = 1 + (int)(blockIdx.y * blockDim.y + threadIdx.y);
        x[0] = 1 + (int)blockIdx.z;
        if (2 * j - 1 > m2 || x[1] > m1) return;
    } else {
        x[0] = 1 + (int)(blockIdx.y * blockDim.y + threadIdx.y);
        if (2 * j - 1 > m1 || x[0] > m0) return;
    }
    const int mL = D == 3 ? m2 : m1;
    const long sL = D == 3 ? s2 : s1;
    int c = 0, b[3] = {0, 0, 0};
#pragma unroll
    for (int a = 0; a < LA; ++a) {
        c |= (x[a] & 1) << (D - 1 - a);
        b[a] = (x[a] + 1) >> 1;
    }
    b[LA] = j;
    const long o = at<D>(L, c, b[0], b[1], b[2]);
    const bool two = 2 * j <= mL;
    const double v1 = src[o + L.cls];  // x = 2j - 1: class bit 1
    const double v0 = two ? src[o] : 0.0;  // x = 2j: class bit 0
    const long so = (long)x[0] * s0 + (D == 3 ? (long)x[1] * s1 : 0) + (long)(2 * j - 1) * sL;
    dst[so] = v1;
    if (two) dst[so + sL] = v0;
}

// launch geometry of k_pack / k_unpack over an (n0, n1[, n2]) box: x over
// PAIRS of the contiguous axis
static inline void pack_grid(int dim, int n0, int n1, int n2, dim3& grd, dim3& blk) {
    blk = dim3(128, 2, 1);
    if (dim == 3) grd = dim3(((n2 + 1) / 2 + 127) / 128, (n1 + 1) / 2, n0);
    else grd = dim3(((n1 + 1) / 2 + 127) / 128, (n0 + 1) / 2, 1);
}

static inline int nb(long n, int t) { return (int)((n + t - 1) / t); }

// ------------------------------------------------------- slab exchanges
// Copy the interior (b1, b2) of plane `sp` of the classes in `mask` from a
// local level array to plane `dp` of a peer's array of the same level
// geometry (peer memory mapped over NVLink P2P / CUDA IPC, or the same
// device for virtual ranks), then fence at system scope so a following
// signal publishes the data.
template <int D>
__global__ void k_push_plane(const double* __restrict__ src, double* __restrict__ dst, Lvl Ls,
                             Lvl Ld, int sp, int dp, unsigned mask) {
    const long n1 = L_B1<D>(Ls), n2 = D == 3 ? Ls.B[2] : 1;
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (!((mask >> c) & 1u) || t >= n1 * n2) return;
    const int b1 = 1 + (int)(t / n2), b2 = D == 3 ? 1 + (int)(t % n2) : 0;
    const double v = src[at<D>(Ls, c, sp, b1, b2)];
    dst[at<D>(Ld, c, dp, b1, b2)] = v;
    __threadfence_system();
}

// Copy planes off+1..off+cnt of every class of a replicated (full) level
// array into the same planes of a peer's copy (the coarse-level gather).
template <int D>
__global__ void k_push_part(const double* __restrict__ src, double* __restrict__ dst, Lvl L,
                            int off, int cntp) {
    const long n1 = L.B[1], n2 = D == 3 ? L.B[2] : 1;
    const long per = n1 * n2;
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (t >= per * cntp) return;
    const int p = off + 1 + (int)(t / per);
    const long r = t % per;
    const int b1 = 1 + (int)(r / n2), b2 = D == 3 ? 1 + (int)(r % n2) : 0;
    const long o = at<D>(L, c, p, b1, b2);
    dst[o] = src[o];
    __threadfence_system();
}

// single-thread publish: bump my send counter for `peer` and store it into
// the peer's arrival slot for me (release, system scope)
__global__ void k_signal(long long* __restrict__ peer_slot, long long* __restrict__ send_cnt) {
    if (threadIdx.x | blockIdx.x) return;
    const long long v = *send_cnt + 1;
    *send_cnt = v;
    __threadfence_system();
    asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(peer_slot), "l"(v) : "memory");
}

// single-thread wait until the arrival counter from a peer reaches the next
// expected value (acquire, system scope)
__global__ void k_wait(const long long* __restrict__ my_slot, long long* __restrict__ expect) {
    if (threadIdx.x | blockIdx.x) return;
    const long long e = *expect + 1;
    *expect = e;
    long long v;
    const long long t0 = clock64();
    do {
        asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(my_slot) : "memory");
        // a peer that never arrives is a protocol bug: fail loudly (~30 s)
        // instead of hanging the device
        if (clock64() - t0 > 60000000000LL) asm volatile("trap;");
        if (v < e) __nanosleep(100);  // back off: keep the memory system free for the peers
    } while (v < e);
    __threadfence_system();
}

// residual partial of this rank (dsum) -> every rank's allpart[rank]
__global__ void k_put_partial(const double* __restrict__ dsum, double* __restrict__ dst) {
    if (threadIdx.x | blockIdx.x) return;
    *dst = *dsum;
    __threadfence_system();
}

// fixed rank-order sum of the partials (identical on every rank)
__global__ void k_sum_partials(const double* __restrict__ allpart, int n, double* out) {
    if (threadIdx.x | blockIdx.x) return;
    double s = allpart[0];
    for (int r = 1; r < n; ++r) s = ad(s, allpart[r]);
    *out = s;
}

// ===========================================================================
// Host engine
// ===========================================================================
// Level arrays shared by engines that never run concurrently (the four
// solves of a projection step run one after another on one stream): the
// i-th array a level requests is the same buffer in every engine bound to
// the arena.  An engine that finds another engine was the last user clears
// all its arrays on load, i.e. starts from the state of a fresh engine.
struct Arena {
    int refs = 1;
    const void* last = nullptr;
    std::map<std::pair<int, int>, std::pair<size_t, double*>> buf;
};
static thread_local Arena* t_arena = nullptr;  // set by fasmg_engine_create_in

struct Engine {
    int dim, ea, nl, s;
    Lvl L[32];
    double* P[32] = {};
    double* F[32] = {};
    double* R[32] = {};
    double* PI[32] = {};
    double* part = nullptr;
    double* dsum = nullptr;  // device scalar
    double* hsum = nullptr;  // pinned host scalar
    int npart = 0;
    BcSpec bc, bch;
    std::vector<unsigned> masks;  // per smoothing step, class masks in order
    cudaStream_t stream = nullptr;
    // V-cycle graphs [starts from a pending speculative half-sweep][with norm]
    cudaGraph_t graphs[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    cudaGraphExec_t execs[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    long kernels_per_vcycle = 0;
    long kernels_per_vcycle_norm = 0;
    long kernels_per_solve_iter = 0;    // a device-loop iteration in steady state (k_conv included)
    // 0: thread per block, 1: per (block, class), 2: 2.5D register march,
    // 3: 2.5D shared-memory march (cp.async) for large 3D levels, 4: the
    // same march fed by TMA boxes (default), else 0
    int sweep_variant = 4;
    int march_chunk = 0;    // planes per marching chunk (0: per-level default)
    int norm_smem = 0;      // dynamic smem of the outer-norm march (FASMG_NORM_SMEM caps CTAs/SM)
    int sweep_minb = 3;     // min resident CTAs of the 3D half-sweep (register cap)
    int edge_fast = 1;      // FASMG_EDGE_FAST: pad-materialised edge transfers (0: ghost chains)
    // ---- axis-0 slab decomposition (multi-GPU / virtual ranks) ----
    int nranks = 1, rank = 0;
    int kg = 0;                         // first replicated level (levels < kg are slabs)
    long long* flags = nullptr;         // [nranks] arrival counters written by peers
    long long* cnt = nullptr;           // [2*nranks] send counters, then expected counters
    double* allpart = nullptr;          // [nranks] residual partial sums, written by peers
    struct Peer {                       // device pointers of every rank, valid in this process
        double* P[32];
        double* F[32];
        double* R[32];                  // edge residual arrays (null for cell fields)
        long long* flags;
        double* allpart;
    };
    std::vector<Peer> peers;            // size nranks once connected
    Arena* arena = nullptr;             // shared level arrays (nullptr: private)
    std::vector<void*> owned;           // level arrays this engine frees
    bool sharded(int k) const { return nranks > 1 && k < kg; }
    bool tma_ok[32] = {};               // level k half-sweeps use k_sweep_tma
    CUtensorMap mapF[32], mapT[32];
    int resid_tma = 1;                  // FASMG_RESID_TMA: tau / norm on the TMA march
    int corr_fuse = 1;                  // FASMG_CORR_FUSE: correction fused into the first post half-sweep
    // ---- the next V-cycle's first half-sweep folded into the outer norm ----
    int spec = 1;                       // FASMG_SPEC (0: off)
    bool spec_ok = false;               // 3D cell unsharded TMA finest level, X plan, no periodic face
    bool spec_pending = false;          // P2 holds X_new of the next V-cycle's first half-sweep
    bool cap_pending = false, cap_spec = false;  // the variant being captured / launched
    bool opp_p2 = false;                // this launch reads the opposite classes from P2
    double* P2 = nullptr;               // finest level, speculative X classes (+ their pads)
    CUtensorMap mapT2;                  // P2 boxes 36 x 10
    // ---- the whole solve as one graph launch (device-side convergence test) ----
    cudaGraph_t gsolve[2] = {nullptr, nullptr};        // [starts from a pending speculation]
    cudaGraphExec_t xsolve[2] = {nullptr, nullptr};
    double* dhist = nullptr;            // residual history (device), SOLVE_CAP entries
    int* dit = nullptr;                 // V-cycles run (device)
    double* dctl = nullptr;             // {tol, scale, k_max} (device)
    double* hbuf = nullptr;             // pinned: ctl (3) + history (SOLVE_CAP) + count
    int corr_chunk = 0;                 // FASMG_CORR_CHUNK: planes per CTA of that sweep (0: march chunk)
    int num_sms = 148;
    int tau_chunk = 0, norm_chunk = 0;  // FASMG_TAU_CHUNK / FASMG_NORM_CHUNK (0: 4 planes)
    int chunk_l1 = 2;                   // FASMG_CHUNK_L1: TMA sweep chunk on levels >= 1 (2: twice
                                        // the CTAs of 4 -- a shorter tail, 38.5 -> 38.0 us at 256^3)
    int edge_tau = 1;                   // FASMG_EDGE_TAU: edge-field tau pass in one march (k_tau_edge_tma)
    int resid_pf = 1;                   // FASMG_RESID_PF: tau/norm marches load f and the axis-0 plane a step ahead
    int etau_chunk = 8;                 // FASMG_ETAU_CHUNK: its planes per CTA
    int fuse_push = 1;                  // FASMG_FUSE_PUSH: sweeps store boundary planes into peers' halos
    // ---- coarse levels in one cluster launch (fasmg_coarse.cuh) ----
    int coarse_k0 = -1;                 // first level run by k_coarse_cycle (-1: none)
    int coarse_cs = 8;                  // FASMG_COARSE_CS: CTAs per cluster
    long coarse_max = 4096;             // FASMG_COARSE_MAX: max blocks of a coarse level
    CoarseArgs* dcoarse = nullptr;      // device copy of the level table
};

struct Tile {
    dim3 grid, block;
};

// tau / outer norm of level k on the TMA march (cell-centred, unsharded)
// level array number idx of level k: the arena's buffer, or a private one
static int lvl_alloc(Engine& E, int k, int idx, size_t bytes, double** out) {
    if (E.arena) {
        auto& slot = E.arena->buf[{k, idx}];
        if (!slot.second) {
            if (int st = fasmg_check(cudaMalloc(&slot.second, bytes))) return st;
            slot.first = bytes;
        }
        if (slot.first >= bytes) {
            *out = slot.second;
            return 0;
        }
    }
    if (int st = fasmg_check(cudaMalloc(out, bytes))) return st;
    E.owned.push_back(*out);
    return 0;
}

// (slab levels too: the axis-0 neighbour planes are the halo planes the
// sweeps keep current, and the coarse writes use global indices)
static bool resid_tma_level(const Engine& E, int k) {
    return E.resid_tma && E.dim == 3 && E.ea < 0 && E.tma_ok[k];
}

// level k's coarse correction rides on its first post-smoothing half-sweep
// (k_sweep_tma<.., CORR>): 3D cell-centred TMA level, unsharded, no periodic
// face, first two half-sweeps complementary X/RBGS color groups
static bool corr_fused(const Engine& E, int k) {
    if (!E.corr_fuse || E.dim != 3 || E.ea >= 0 || !E.tma_ok[k] || E.sharded(k) ||
        k + 1 >= E.nl || !E.PI[k + 1] || E.masks.size() < 2 || 8 * E.L[k + 1].cls >= INT_MAX)
        return false;  // (the kernel addresses the coarse level with 32-bit offsets)
    for (int a = 0; a < 3; ++a)
        if (E.bc.kind[a][0] == BC_PERIODIC || E.bc.kind[a][1] == BC_PERIODIC) return false;
    const unsigned m0 = E.masks[0], m1 = E.masks[1];
    return (m0 == 0x96u || m0 == 0x69u) && m1 == (m0 ^ 0xFFu);
}

// edge fields: level k's correction (prolongation of Corr) rides on the
// first post-smoothing half-sweep (k_sweep_tma<EA, M, true>): the same plan
// and boundary conditions as corr_fused, the edge_fast transfers
static bool ecorr_fused(const Engine& E, int k) {
    if (!E.corr_fuse || E.dim != 3 || E.ea < 0 || !E.edge_fast || !E.tma_ok[k] ||
        E.sharded(k) || k + 1 >= E.nl || E.masks.size() < 2 || 8 * E.L[k + 1].cls >= INT_MAX)
        return false;
    for (int a = 0; a < 3; ++a)
        if (E.bc.kind[a][0] == BC_PERIODIC || E.bc.kind[a][1] == BC_PERIODIC) return false;
    const unsigned m0 = E.masks[0], m1 = E.masks[1];
    return (m0 == 0x96u || m0 == 0x69u) && m1 == (m0 ^ 0xFFu);
}

// level k's edge-field tau pass runs as one TMA march (k_tau_edge_tma):
// 3D edge field, unsharded TMA level, no periodic face
static bool edge_tau_level(const Engine& E, int k) {
    if (!E.edge_tau || E.dim != 3 || E.ea < 0 || !E.tma_ok[k] || E.sharded(k) || k + 1 >= E.nl)
        return false;
    for (int a = 0; a < 3; ++a)
        if (E.bc.kind[a][0] == BC_PERIODIC || E.bc.kind[a][1] == BC_PERIODIC) return false;
    return true;
}

static dim3 resid_grid(const Lvl& L, int chunk) {
    using namespace rsw;
    return dim3((L.B[2] + TX - 1) / TX, (L.B[1] + TY - 1) / TY, (L.B[0] + chunk - 1) / chunk);
}

static unsigned p2ceil(unsigned v) {
    unsigned r = 1;
    while (r < v) r <<= 1;
    return r;
}

// thread block shape over (b2, b1, b0) [3D] or (b1, b0) [2D]
static unsigned g_tile_y = 8;  // FASMG_TILE_Y: rows of b1 per CTA (3D)

static Tile tile_of(const Lvl& L) {
    Tile t;
    if (L.dim == 3) {
        unsigned bx = std::min(32u, p2ceil(L.B[2]));
        unsigned by = std::min(std::min(g_tile_y, 256u / bx), p2ceil(L.B[1]));
        unsigned bz = std::min(256u / (bx * by), p2ceil(L.B[0]));
        t.block = dim3(bx, by, bz);
        t.grid = dim3((L.B[2] + bx - 1) / bx, (L.B[1] + by - 1) / by, (L.B[0] + bz - 1) / bz);
    } else {
        unsigned bx = std::min(64u, p2ceil(L.B[1]));
        unsigned by = std::min(256u / bx, p2ceil(L.B[0]));
        t.block = dim3(bx, by, 1);
        t.grid = dim3((L.B[1] + bx - 1) / bx, (L.B[0] + by - 1) / by, 1);
    }
    return t;
}

static inline long tile_ctas(const Tile& t) { return (long)t.grid.x * t.grid.y * t.grid.z; }

// class masks the sweep kernel is instantiated for: all odd / all even
// index-sum classes (X and RBGS plans) and single classes (U/Z plans)
static bool mask_supported(int dim, unsigned m) {
    unsigned odd = dim == 3 ? 0x96u : 0x6u, even = dim == 3 ? 0x69u : 0x9u;
    if (m == odd || m == even) return true;
    return m != 0 && (m & (m - 1)) == 0 && m < (1u << (1 << dim));
}

// the neighbours' halo planes for a fused push (sharded levels only)
static PeerHalo peer_halo(const Engine& E, int k) {
    PeerHalo ph;
    if (!E.fuse_push || !E.sharded(k)) return ph;
    if (E.rank > 0) ph.lo = E.peers[E.rank - 1].P[k];
    if (E.rank + 1 < E.nranks) ph.hi = E.peers[E.rank + 1].P[k];
    return ph;
}

// returns true when the kernel also pushed the updated boundary planes
template <int D, int EA, unsigned M>
static bool sweep_one(Engine& E, int k, const Tile& t) {
    const Lvl& L = E.L[k];
    const PeerHalo ph = peer_halo(E, k);
    const bool fused = ph.lo || ph.hi;
    if (E.sweep_variant == 1) {
        constexpr int NCM = __builtin_popcount(M);
        dim3 blk, grd;
        if (D == 3) {
            unsigned bx = std::min(32u, p2ceil(L.B[2]));
            unsigned by = std::min(256u / bx, p2ceil(L.B[1]));
            blk = dim3(bx, by, 1);
            grd = dim3((L.B[2] + bx - 1) / bx, (L.B[1] + by - 1) / by, L.B[0] * NCM);
        } else {
            unsigned bx = std::min(64u, p2ceil(L.B[1]));
            unsigned by = std::min(256u / bx, p2ceil(L.B[0]));
            blk = dim3(bx, by, 1);
            grd = dim3((L.B[1] + bx - 1) / bx, (L.B[0] + by - 1) / by, NCM);
        }
        k_sweep_pc<D, EA, M><<<grd, blk, 0, E.stream>>>(E.P[k], E.F[k], L, E.bc);
        return false;
    }
    if (E.sweep_variant == 2 && __builtin_popcount(M) > 1) {
        const int chunk = E.march_chunk > 0 ? E.march_chunk : 16;
        dim3 blk, grd;
        const unsigned nch = (L.B[0] + chunk - 1) / chunk;
        if (D == 3) {
            unsigned bx = std::min(32u, p2ceil(L.B[2]));
            unsigned by = std::min(256u / bx, p2ceil(L.B[1]));
            blk = dim3(bx, by, 1);
            grd = dim3((L.B[2] + bx - 1) / bx, (L.B[1] + by - 1) / by, nch);
        } else {
            unsigned bx = std::min(256u, p2ceil(L.B[1]));
            blk = dim3(bx, 1, 1);
            grd = dim3((L.B[1] + bx - 1) / bx, nch, 1);
        }
        k_sweep_march<D, EA, M><<<grd, blk, 0, E.stream>>>(E.P[k], E.F[k], L, E.bc, chunk);
        return false;
    }
    if (D == 2 && E.sweep_variant == 4 && E.tma_ok[k] && __builtin_popcount(M) > 1) {
        using namespace tsw2;
        const int steps = E.march_chunk > 0 ? E.march_chunk : 4;
        dim3 blk(TX, TY, 1);
        dim3 grd((L.B[1] + TX - 1) / TX, (L.B[0] + steps * TY - 1) / (steps * TY), 1);
        k_sweep_tma2d<EA, M><<<grd, blk, SMEM, E.stream>>>(E.mapT[k], E.mapF[k], E.P[k], L,
                                                           E.bc, steps, ph);
        return fused;
    }
    if (D == 3 && E.sweep_variant == 4 && E.tma_ok[k] && __builtin_popcount(M) > 1) {
        using namespace tsw;
        // 4-plane chunks: 16384 CTAs at 512^3; the 2 window planes a chunk
        // re-loads are L2 hits of the neighbouring chunk's CTAs (ncu: 1.63 GB
        // per finest launch vs 1.69 GB at 16 planes), and the many short
        // CTAs keep every SM's TMA queue full to the end of the launch:
        // 276 -> 248 us (B200, profiles/r01g_ncu_summary.txt)
        const int chunk = E.march_chunk > 0 ? E.march_chunk : (k > 0 && E.chunk_l1 > 0 ? E.chunk_l1 : 4);
        dim3 blk(TX, TY, 1);
        dim3 grd((L.B[2] + TX - 1) / TX, (L.B[1] + TY - 1) / TY, (L.B[0] + chunk - 1) / chunk);
        k_sweep_tma<EA, M><<<grd, blk, SMEM, E.stream>>>(E.opp_p2 && k == 0 ? E.mapT2 : E.mapT[k],
                                                         E.mapF[k], E.P[k], L, E.bc,
                                                         chunk, nullptr, nullptr, Lvl(), ph);
        return fused;
    }
    if (D == 3 && E.sweep_variant >= 3 && __builtin_popcount(M) > 1 && L.B[2] >= 32 &&
        L.B[1] >= 8 && L.nblk >= (1L << 21)) {
        using namespace smem_sweep;
        // planes per marching chunk: long chunks amortize the two window
        // planes each chunk loads twice; short ones keep >= 8 CTAs per SM
        // in flight (B200 measurements: 16 at 256 planes, 4 at 128)
        const long tiles = (long)((L.B[2] + TX - 1) / TX) * ((L.B[1] + TY - 1) / TY);
        int chunk = E.march_chunk;
        if (chunk <= 0) {
            chunk = 4;
            for (int c = 16; c >= 8; c >>= 1)
                if (tiles * ((L.B[0] + c - 1) / c) >= 1184) { chunk = c; break; }
        }
        dim3 blk(TX, TY, 1);
        dim3 grd((L.B[2] + TX - 1) / TX, (L.B[1] + TY - 1) / TY, (L.B[0] + chunk - 1) / chunk);
        const size_t shm = sizeof(double) * 4 * RING * PL;
        k_sweep_smem<EA, M><<<grd, blk, shm, E.stream>>>(E.P[k], E.F[k], L, E.bc, chunk);
        return false;
    }
    if (D == 3 && E.sweep_minb == 4 && __builtin_popcount(M) > 1)
        k_sweep_fast<D, EA, M, 4><<<t.grid, t.block, 0, E.stream>>>(E.P[k], E.F[k], L, E.bc, ph);
    else
        k_sweep_fast<D, EA, M><<<t.grid, t.block, 0, E.stream>>>(E.P[k], E.F[k], L, E.bc, ph);
    return fused;
}

template <int D, int EA>
static bool sweep_mask(Engine& E, int k, unsigned m, const Tile& t) {
    if (D == 3) {
        switch (m) {
            case 0x96u: return sweep_one<D, EA, 0x96u>(E, k, t);
            case 0x69u: return sweep_one<D, EA, 0x69u>(E, k, t);
            case 0x01u: return sweep_one<D, EA, 0x01u>(E, k, t);
            case 0x02u: return sweep_one<D, EA, 0x02u>(E, k, t);
            case 0x04u: return sweep_one<D, EA, 0x04u>(E, k, t);
            case 0x08u: return sweep_one<D, EA, 0x08u>(E, k, t);
            case 0x10u: return sweep_one<D, EA, 0x10u>(E, k, t);
            case 0x20u: return sweep_one<D, EA, 0x20u>(E, k, t);
            case 0x40u: return sweep_one<D, EA, 0x40u>(E, k, t);
            case 0x80u: return sweep_one<D, EA, 0x80u>(E, k, t);
        }
    } else {
        switch (m) {
            case 0x6u: return sweep_one<D, EA, 0x6u>(E, k, t);
            case 0x9u: return sweep_one<D, EA, 0x9u>(E, k, t);
            case 0x1u: return sweep_one<D, EA, 0x1u>(E, k, t);
            case 0x2u: return sweep_one<D, EA, 0x2u>(E, k, t);
            case 0x4u: return sweep_one<D, EA, 0x4u>(E, k, t);
            case 0x8u: return sweep_one<D, EA, 0x8u>(E, k, t);
        }
    }
    return false;
}

// dispatch the runtime edge axis onto the compile-time one
#define EA_DISPATCH(D, EAV, CALL)                              \
    do {                                                       \
        switch (EAV) {                                         \
            case -1: { constexpr int EA = -1; CALL; } break;   \
            case 0: { constexpr int EA = 0; CALL; } break;     \
            case 1: { constexpr int EA = 1; CALL; } break;     \
            default: { constexpr int EA = (D == 3 ? 2 : 1); CALL; } break; \
        }                                                      \
    } while (0)

// grid of a per-face kernel over (n1 x n2) face positions per face (the
// largest over the faces), z = nz face slots
template <int D>
static dim3 face_grid(const int* ext, int nz, int tpb) {
    int n1 = 1, n2 = 1;  // first / last other axis, maximised over the faces
    for (int a = 0; a < D; ++a) {
        int oth[2], no = 0;
        for (int t = 0; t < D; ++t)
            if (t != a) oth[no++] = t;
        if (D == 3) {
            n1 = std::max(n1, ext[oth[0]]);
            n2 = std::max(n2, ext[oth[1]]);
        } else {
            n2 = std::max(n2, ext[oth[0]]);
        }
    }
    return dim3((n2 + tpb - 1) / tpb, n1, nz);
}

template <int D>
static void launch_pad_fill(Engine& E, int k, long& cnt) {
    const Lvl& L = E.L[k];
    const dim3 grid = face_grid<D>(L.B, 2 * D, 128);
    EA_DISPATCH(D, E.ea, (k_pad_fill<D, EA><<<grid, 128, 0, E.stream>>>(E.P[k], L, E.bc)));
    ++cnt;
}

template <int D>
static void launch_pad_all(Engine& E, double* P, const Lvl& L, const BcSpec& bc, long& cnt) {
    k_pad_all<D><<<face_grid<D>(L.E, 2 * D, TPB), TPB, 0, E.stream>>>(P, L, bc);
    ++cnt;
}

template <int D>
static void launch_pad_all2(Engine& E, int k, long& cnt) {
    const Lvl& L = E.L[k];
    k_pad_all2<D><<<face_grid<D>(L.E, 4 * D, TPB), TPB, 0, E.stream>>>(E.P[k], E.bc, E.R[k],
                                                                        E.bch, L);
    ++cnt;
}

// ---- slab exchanges (no-ops on a single rank) ----
// pushed: the sweep kernel already stored the planes into the peers (fused
// push) -- only the counters are published
// arr: 0 the level's P arrays, 1 its R arrays (edge residual, whose
// restriction reads the halo plane when axis 0 is tangential)
template <int D>
static void halo_exchange(Engine& E, int k, unsigned mask, long& cnt, bool pushed = false,
                          int arr = 0) {
    if (!E.sharded(k)) return;
    double* mine = arr ? E.R[k] : E.P[k];
    auto theirs = [&](int q) { return arr ? E.peers[q].R[k] : E.peers[q].P[k]; };
    const Lvl& L = E.L[k];
    const int r = E.rank, P = E.nranks;
    const unsigned bit0 = 1u << (D - 1);
    unsigned up = 0, dn = 0;  // q0=0 classes feed the upper neighbor's lower halo
    for (int c = 0; c < (1 << D); ++c)
        if ((mask >> c) & 1u) {
            if (c & bit0) dn |= 1u << c;
            else up |= 1u << c;
        }
    const long n = (long)L.B[1] * (D == 3 ? L.B[2] : 1);
    const dim3 grid(nb(n, TPB), 1 << D);
    if (r + 1 < P && up) {
        if (!pushed) {
            k_push_plane<D><<<grid, TPB, 0, E.stream>>>(mine, theirs(r + 1), L, L, L.B[0], 0, up);
            ++cnt;
        }
        k_signal<<<1, 1, 0, E.stream>>>(E.peers[r + 1].flags + r, E.cnt + (r + 1));
        ++cnt;
    }
    if (r > 0 && dn) {
        if (!pushed) {
            k_push_plane<D><<<grid, TPB, 0, E.stream>>>(mine, theirs(r - 1), L, L, 1, L.B[0] + 1,
                                                         dn);
            ++cnt;
        }
        k_signal<<<1, 1, 0, E.stream>>>(E.peers[r - 1].flags + r, E.cnt + (r - 1));
        ++cnt;
    }
    if (r > 0 && up) {
        k_wait<<<1, 1, 0, E.stream>>>(E.flags + (r - 1), E.cnt + P + (r - 1));
        ++cnt;
    }
    if (r + 1 < P && dn) {
        k_wait<<<1, 1, 0, E.stream>>>(E.flags + (r + 1), E.cnt + P + (r + 1));
        ++cnt;
    }
}

// Data-free handshake with both neighbours.  Needed where a halo that was
// just read in full (by the coarse source term) would otherwise be
// overwritten by a neighbour's next push before the read finished: the
// first smoothing half-sweep of a sharded coarse level pushes classes that
// coarse_src still reads (write-after-read across ranks).
static void neighbor_barrier(Engine& E, int k, long& cnt) {
    if (!E.sharded(k)) return;
    const int r = E.rank, P = E.nranks;
    for (int q : {r - 1, r + 1}) {
        if (q < 0 || q >= P) continue;
        k_signal<<<1, 1, 0, E.stream>>>(E.peers[q].flags + r, E.cnt + q);
        ++cnt;
    }
    for (int q : {r - 1, r + 1}) {
        if (q < 0 || q >= P) continue;
        k_wait<<<1, 1, 0, E.stream>>>(E.flags + q, E.cnt + P + q);
        ++cnt;
    }
}

// level kg is replicated: every rank pushes the coarse planes its slab of
// level kg-1 produced (P and F) into every peer's copy, then pads are filled
template <int D>
static void gather_level(Engine& E, int k, long& cnt) {
    const Lvl& L = E.L[k];
    const int P = E.nranks, r = E.rank;
    const int part = L.B[0] / P;  // coarse planes per rank (whole blocks: fine nb even)
    const int off = r * part;
    const long n = (long)L.B[1] * (D == 3 ? L.B[2] : 1) * part;
    const dim3 grid(nb(n, TPB), 1 << D);
    for (int q = 0; q < P; ++q) {
        if (q == r) continue;
        k_push_part<D><<<grid, TPB, 0, E.stream>>>(E.P[k], E.peers[q].P[k], L, off, part);
        k_push_part<D><<<grid, TPB, 0, E.stream>>>(E.F[k], E.peers[q].F[k], L, off, part);
        k_signal<<<1, 1, 0, E.stream>>>(E.peers[q].flags + r, E.cnt + q);
        cnt += 3;
    }
    for (int q = 0; q < P; ++q) {
        if (q == r) continue;
        k_wait<<<1, 1, 0, E.stream>>>(E.flags + q, E.cnt + P + q);
        ++cnt;
    }
    launch_pad_fill<D>(E, k, cnt);
}

template <int A>
static void launch_sweep_ecorr(Engine& E, int k, unsigned m, dim3 grd, dim3 blk, int chunk) {
    using namespace tsw;
    if (m == 0x96u)
        k_sweep_tma<A, 0x96u, true><<<grd, blk, SMEM_ECORR, E.stream>>>(
            E.mapT[k], E.mapF[k], E.P[k], E.L[k], E.bc, chunk, E.R[k + 1], nullptr, E.L[k + 1],
            PeerHalo(), E.F[k]);
    else
        k_sweep_tma<A, 0x69u, true><<<grd, blk, SMEM_ECORR, E.stream>>>(
            E.mapT[k], E.mapF[k], E.P[k], E.L[k], E.bc, chunk, E.R[k + 1], nullptr, E.L[k + 1],
            PeerHalo(), E.F[k]);
}

// the first post-smoothing half-sweep of level k with the coarse correction
// applied on the fly (k_sweep_tma<-1, M, true>; see corr_fused)
static void launch_sweep_corr(Engine& E, int k, unsigned m) {
    using namespace tsw;
    const Lvl& L = E.L[k];
    const Lvl& Lc = E.L[k + 1];
    // (longer chunks amortize the per-chunk prologue of the correction
    // ring -- for edge fields also of the box correction -- as long as the
    // grid keeps >= 4 waves of 3 CTAs per SM)
    int chunk = E.corr_chunk > 0 ? E.corr_chunk : (E.march_chunk > 0 ? E.march_chunk : 4);
    if (E.corr_chunk <= 0 && E.march_chunk <= 0) {
        const long plane = (long)((L.B[2] + TX - 1) / TX) * ((L.B[1] + TY - 1) / TY);
        for (int c = E.ea >= 0 ? 16 : 8; c > 4; c >>= 1)
            if (plane * ((L.B[0] + c - 1) / c) >= 4L * 3 * E.num_sms) { chunk = c; break; }
    }
    dim3 blk(TX, TY, 1);
    dim3 grd((L.B[2] + TX - 1) / TX, (L.B[1] + TY - 1) / TY, (L.B[0] + chunk - 1) / chunk);
    if (E.ea >= 0) {  // edge: Pc = the coarse Corr array (k_corr_edge_*)
        EA_DISPATCH(3, E.ea, (launch_sweep_ecorr<(EA < 0 ? 0 : EA)>(E, k, m, grd, blk, chunk)));
    } else if (m == 0x96u)
        k_sweep_tma<-1, 0x96u, true><<<grd, blk, SMEM_CORR, E.stream>>>(
            E.mapT[k], E.mapF[k], E.P[k], L, E.bc, chunk, E.P[k + 1], E.PI[k + 1], Lc, PeerHalo(),
            E.F[k]);
    else
        k_sweep_tma<-1, 0x69u, true><<<grd, blk, SMEM_CORR, E.stream>>>(
            E.mapT[k], E.mapF[k], E.P[k], L, E.bc, chunk, E.P[k + 1], E.PI[k + 1], Lc, PeerHalo(),
            E.F[k]);
}

// spec_start: the previous outer norm already ran this stage's first
// launch into P2 (k_resid_tma<2>): skip it, and let the second launch read
// its opposite classes from P2
template <int D>
static void launch_smooth(Engine& E, int k, long& cnt, bool first_corr = false,
                          bool spec_start = false) {
    const Tile t = tile_of(E.L[k]);
    for (int it = 0; it < E.s; ++it)
        for (int jm = 0; jm < (int)E.masks.size(); ++jm) {
            const unsigned m = E.masks[jm];
            if (spec_start && it == 0 && jm == 0) continue;
            E.opp_p2 = spec_start && it == 0 && jm == 1;
            bool pushed = false;
            if (first_corr && it == 0 && m == E.masks[0]) {
                launch_sweep_corr(E, k, m);
                first_corr = false;
            } else {
                EA_DISPATCH(D, E.ea, (pushed = sweep_mask<D, EA>(E, k, m, t)));
            }
            E.opp_p2 = false;
            ++cnt;
            halo_exchange<D>(E, k, m, cnt, pushed);
        }
}

template <int D>
static void launch_coarse(Engine& E, long& cnt) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(E.coarse_cs, 1, 1);
    cfg.blockDim = dim3(512, 1, 1);
    cfg.stream = E.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = E.coarse_cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_coarse_cycle<D>, (const CoarseArgs*)E.dcoarse);
    ++cnt;
}

template <int D>
static void launch_vcycle(Engine& E, long& cnt) {
    const unsigned ALL = (1u << (1 << D)) - 1;
    // levels >= kc run inside one cluster launch
    const int kc = E.coarse_k0 >= 0 ? E.coarse_k0 : E.nl;
    if (kc == 0) {
        launch_coarse<D>(E, cnt);
        return;
    }
    // descent
    for (int k = 0; k < std::min(kc, E.nl - 1); ++k) {
        const Lvl& L = E.L[k];
        const Lvl& Lc = E.L[k + 1];
        const Tile t = tile_of(L), tc = tile_of(Lc);
        launch_smooth<D>(E, k, cnt, false, D == 3 && k == 0 && E.cap_pending);
        if (E.ea < 0) {
            {
                if (D == 3 && resid_tma_level(E, k)) {
                    const int ch = E.march_chunk > 0 ? E.march_chunk : (E.tau_chunk > 0 ? E.tau_chunk : 4);
                    if (E.resid_pf)
                        k_resid_tma<1, -1, true><<<resid_grid(L, ch), dim3(rsw::TX, rsw::TY, 1),
                                                   rsw::SMEM, E.stream>>>(
                            E.mapT[k], E.P[k], E.F[k], L, E.bc, ch, nullptr, E.P[k + 1],
                            E.F[k + 1], Lc, corr_fused(E, k) ? E.PI[k + 1] : nullptr);
                    else
                    k_resid_tma<1><<<resid_grid(L, ch), dim3(rsw::TX, rsw::TY, 1), rsw::SMEM,
                                     E.stream>>>(E.mapT[k], E.P[k], E.F[k], L, E.bc, ch,
                                                 nullptr, E.P[k + 1], E.F[k + 1], Lc,
                                                 corr_fused(E, k) ? E.PI[k + 1] : nullptr);
                } else {
                    k_tau_fast<D><<<t.grid, t.block, 0, E.stream>>>(
                        E.P[k], E.F[k], L, E.P[k + 1], E.F[k + 1], Lc, E.bc,
                        corr_fused(E, k) ? E.PI[k + 1] : nullptr);
                }
                ++cnt;
            }
        } else if (D == 3 && edge_tau_level(E, k)) {
            const int ch = E.etau_chunk;
            EA_DISPATCH(3, E.ea, (k_tau_edge_tma<(EA < 0 ? 0 : EA)><<<resid_grid(L, ch),
                                       dim3(esw::TX, esw::TY, 1), esw::SMEM, E.stream>>>(
                                     E.mapT[k], E.P[k], E.F[k], L, E.bc, E.bch, ch, E.P[k + 1],
                                     E.F[k + 1], Lc, E.PI[k + 1])));
            ++cnt;
            launch_pad_fill<D>(E, k + 1, cnt);
        } else {
            long mc = 1;
            for (int a = 0; a < D; ++a) {
                const long ma = a == E.ea ? Lc.n[a] - 1 : Lc.n[a];
                mc *= a == 0 ? restrict_rows(L, ma) : ma;
            }
            EA_DISPATCH(D, E.ea, (k_residual_fast<D, EA><<<t.grid, t.block, 0, E.stream>>>(
                                     E.P[k], E.F[k], E.R[k], L)));
            // tangential axis 0: the restriction of r reads the upper halo plane
            if (E.ea != 0) halo_exchange<D>(E, k, ALL, cnt, false, 1);
            if (E.edge_fast) {
                launch_pad_all2<D>(E, k, cnt);
                EA_DISPATCH(D, E.ea, (k_restrict_edge_fast<D, EA><<<nb(mc, TPB), TPB, 0,
                                                                    E.stream>>>(E.P[k], L,
                                                                                E.P[k + 1], Lc)));
                EA_DISPATCH(D, E.ea, (k_restrict_edge_fast<D, EA><<<nb(mc, TPB), TPB, 0,
                                                                    E.stream>>>(E.R[k], L,
                                                                                E.F[k + 1], Lc)));
            } else {
                k_restrict_edge<D><<<nb(mc, TPB), TPB, 0, E.stream>>>(E.P[k], L, E.bc,
                                                                      E.P[k + 1], Lc);
                k_restrict_edge<D><<<nb(mc, TPB), TPB, 0, E.stream>>>(E.R[k], L, E.bch,
                                                                      E.F[k + 1], Lc);
            }
            cnt += 3;
            launch_pad_fill<D>(E, k + 1, cnt);
        }
        if (E.sharded(k + 1)) halo_exchange<D>(E, k + 1, ALL, cnt);
        else if (E.sharded(k)) gather_level<D>(E, k + 1, cnt);
        if (E.ea >= 0 && !(D == 3 && edge_tau_level(E, k))) {  // pinit = R p, copied after the exchange: halo planes too
            const long tot = Lc.cls * (1 << D);
            k_copy_blk<D><<<nb(tot, TPB), TPB, 0, E.stream>>>(E.P[k + 1], E.PI[k + 1], tot);
            ++cnt;
        }
        EA_DISPATCH(D, E.ea, (k_coarse_src_fast<D, EA><<<tc.grid, tc.block, 0, E.stream>>>(
                                 E.P[k + 1], E.F[k + 1], Lc)));
        ++cnt;
        neighbor_barrier(E, k + 1, cnt);
    }
    if (kc < E.nl) launch_coarse<D>(E, cnt);
    else launch_smooth<D>(E, E.nl - 1, cnt);  // coarsest: s smoothing steps
    // ascent
    for (int k = std::min(kc, E.nl - 1) - 1; k >= 0; --k) {
        const Lvl& L = E.L[k];
        const Lvl& Lc = E.L[k + 1];
        const Tile t = tile_of(L);
        const bool cf = D == 3 && (corr_fused(E, k) || ecorr_fused(E, k));  // rides on the first sweep
        if (E.ea < 0) {
            if (!cf) {
                k_correct_fast<D><<<t.grid, t.block, 0, E.stream>>>(E.P[k], L, E.P[k + 1], Lc,
                                                                     E.bc);
                ++cnt;
            }
        } else {
            if (E.edge_fast) {
                dim3 cg, cbk;
                corr_edge_grid<D>(Lc, cg, cbk);
                const Tile tcc = tile_of(Lc);
                k_corr_edge_in<D><<<tcc.grid, tcc.block, 0, E.stream>>>(E.P[k + 1], E.PI[k + 1],
                                                                         Lc, E.R[k + 1]);
                {
                    int mx = 1;
                    for (int a = 0; a < D; ++a) mx = std::max(mx, Lc.E[a]);
                    const dim3 pg((mx + TPB - 1) / TPB, D == 3 ? mx : 1, 2 * D + 1);
                    k_corr_edge_pads<D><<<pg, TPB, 0, E.stream>>>(E.P[k + 1], E.PI[k + 1], Lc,
                                                                  E.bch, E.R[k + 1]);
                }
                cnt += 2;
                if (!cf) {
                    EA_DISPATCH(D, E.ea, (k_correct_edge_fast<D, EA><<<t.grid, t.block, 0,
                                                                       E.stream>>>(E.P[k], L,
                                                                                   E.R[k + 1], Lc)));
                    ++cnt;
                }
            } else {
                k_correct_edge<D><<<nb(L.nblk, TPB), TPB, 0, E.stream>>>(E.P[k], L, E.P[k + 1],
                                                                         E.PI[k + 1], Lc, E.bch);
                ++cnt;
            }
            if (!cf) launch_pad_fill<D>(E, k, cnt);
        }
        halo_exchange<D>(E, k, ALL, cnt);
        launch_smooth<D>(E, k, cnt, cf);
    }
}

template <int D>
static void launch_norm(Engine& E, long& cnt) {
    const Lvl& L = E.L[0];
    const Tile t = tile_of(L);
    int npart_norm = E.npart;
    if (D == 3 && E.cap_spec) {  // norm + the next V-cycle's first half-sweep (into P2)
        const int ch = E.march_chunk > 0 ? E.march_chunk : (E.norm_chunk > 0 ? E.norm_chunk : 4);
        const dim3 g = resid_grid(L, ch), b(rsw::TX, rsw::TY, 1);
        if (E.masks[0] == 0x96u)
            k_resid_tma<2, -1, true, 0x96u><<<g, b, E.norm_smem, E.stream>>>(
                E.mapT[0], E.P[0], E.F[0], L, E.bc, ch, E.part, nullptr, nullptr, L, nullptr,
                E.P2, E.P[0]);
        else
            k_resid_tma<2, -1, true, 0x69u><<<g, b, E.norm_smem, E.stream>>>(
                E.mapT[0], E.P[0], E.F[0], L, E.bc, ch, E.part, nullptr, nullptr, L, nullptr,
                E.P2, E.P[0]);
        npart_norm = (int)(g.x * g.y * g.z);
        ++cnt;
    } else {
        if (D == 3 && E.resid_tma && E.tma_ok[0]) {
            const int ch = E.march_chunk > 0 ? E.march_chunk : (E.norm_chunk > 0 ? E.norm_chunk : 4);
            const dim3 g = resid_grid(L, ch);
            if (E.resid_pf)
                EA_DISPATCH(3, E.ea, (k_resid_tma<0, EA, true><<<g, dim3(rsw::TX, rsw::TY, 1),
                                                                 E.norm_smem, E.stream>>>(
                                         E.mapT[0], E.P[0], E.F[0], L, E.bc, ch, E.part, nullptr,
                                         nullptr, L, nullptr)));
            else
            EA_DISPATCH(3, E.ea, (k_resid_tma<0, EA><<<g, dim3(rsw::TX, rsw::TY, 1), E.norm_smem,
                                                       E.stream>>>(
                                     E.mapT[0], E.P[0], E.F[0], L, E.bc, ch, E.part, nullptr,
                                     nullptr, L, nullptr)));
            npart_norm = (int)(g.x * g.y * g.z);
        } else if (E.ea < 0) {
            // (walking axis 0 in chunks per thread measured slower: 1 block)
            const int ch = 1;
            Tile tt = t;
            if (D == 3) tt.grid.z = (L.B[0] + ch * tt.block.z - 1) / (ch * tt.block.z);
            k_res_sumsq_cell<D><<<tt.grid, tt.block, 0, E.stream>>>(E.P[0], E.F[0], L, E.part,
                                                                     ch);
            npart_norm = (int)tile_ctas(tt);
        } else
            EA_DISPATCH(D, E.ea, (k_res_sumsq_fast<D, EA><<<t.grid, t.block, 0, E.stream>>>(
                                     E.P[0], E.F[0], L, E.part)));
        ++cnt;
    }
    k_final_sum<<<1, 1024, 0, E.stream>>>(E.part, npart_norm, E.dsum);
    ++cnt;
    if (E.nranks > 1) {  // fixed rank-order sum of the partials on every rank
        const int P = E.nranks, r = E.rank;
        for (int q = 0; q < P; ++q) {
            k_put_partial<<<1, 1, 0, E.stream>>>(E.dsum, E.peers[q].allpart + r);
            ++cnt;
            if (q != r) {
                k_signal<<<1, 1, 0, E.stream>>>(E.peers[q].flags + r, E.cnt + q);
                ++cnt;
            }
        }
        for (int q = 0; q < P; ++q)
            if (q != r) {
                k_wait<<<1, 1, 0, E.stream>>>(E.flags + q, E.cnt + P + q);
                ++cnt;
            }
        k_sum_partials<<<1, 1, 0, E.stream>>>(E.allpart, P, E.dsum);
        ++cnt;
    }
}

// capture the V-cycle (+ norm) variant for the current speculation state
static int capture(Engine& E, bool with_norm, cudaGraph_t* g, cudaGraphExec_t* ex) {
    long cnt = 0;
    E.cap_pending = E.spec_ok && E.spec_pending;
    E.cap_spec = E.spec_ok && with_norm;
    cudaError_t e = cudaStreamBeginCapture(E.stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return fasmg_check(e);
    if (E.dim == 3) {
        launch_vcycle<3>(E, cnt);
        if (with_norm) launch_norm<3>(E, cnt);
    } else {
        launch_vcycle<2>(E, cnt);
        if (with_norm) launch_norm<2>(E, cnt);
    }
    if (with_norm) {
        cudaMemcpyAsync(E.hsum, E.dsum, sizeof(double), cudaMemcpyDeviceToHost, E.stream);
    }
    e = cudaStreamEndCapture(E.stream, g);
    if (e != cudaSuccess) return fasmg_check(e);
    e = cudaGraphInstantiate(ex, *g, 0);
    if (e != cudaSuccess) return fasmg_check(e);
    if (!E.cap_pending) {
        if (with_norm) E.kernels_per_vcycle_norm = cnt;
        else E.kernels_per_vcycle = cnt;
    }
    E.cap_pending = E.cap_spec = false;
    return 0;
}

// the graph variant for the current state, and the state after it runs
static void graph_slot(Engine& E, bool with_norm, cudaGraph_t** g, cudaGraphExec_t** ex) {
    const int pi = E.spec_ok && E.spec_pending ? 1 : 0;
    *g = &E.graphs[pi][with_norm ? 1 : 0];
    *ex = &E.execs[pi][with_norm ? 1 : 0];
}
static void after_launch(Engine& E, bool with_norm) { E.spec_pending = E.spec_ok && with_norm; }

// ---------------------------------------------------- device-side solve loop
// FasSolver.solve's outer loop (PKG/fas.py:147-154) with the convergence test
// on the device: after each V-cycle + norm, k_conv forms res = scale *
// sqrt(sumsq) exactly as the host does (IEEE sqrt and multiply), appends it to
// the history and sets the WHILE node's condition to !(res <= tol) && it <
// k_max -- so a whole solve is ONE graph launch, with no host round trip
// between V-cycles, and the same cycles / history / fields as the host loop.
constexpr int SOLVE_CAP = 4096;
__global__ void k_conv(const double* __restrict__ dsum, const double* __restrict__ ctl,
                       double* __restrict__ hist, int* __restrict__ it,
                       cudaGraphConditionalHandle h) {
    const double res = ml(ctl[1], __dsqrt_rn(dsum[0]));
    const int i = it[0];
    hist[i] = res;
    it[0] = i + 1;
    cudaGraphSetConditional(h, (!(res <= ctl[0]) && (double)(i + 1) < ctl[2]) ? 1u : 0u);
}

template <int D>
static void capture_iteration(Engine& E, bool pending, cudaGraphConditionalHandle h) {
    long cnt = 0;
    E.cap_pending = E.spec_ok && pending;
    E.cap_spec = E.spec_ok;
    launch_vcycle<D>(E, cnt);
    launch_norm<D>(E, cnt);
    E.cap_pending = E.cap_spec = false;
    k_conv<<<1, 1, 0, E.stream>>>(E.dsum, E.dctl, E.dhist, E.dit, h);
    if (pending) E.kernels_per_solve_iter = cnt + 1;  // the WHILE body
}

// [first iteration (from the current speculation state)] -> WHILE(cond) {
// iteration (from the pending state the previous one leaves) }
static int build_solve_graph(Engine& E, int ps) {
    cudaGraph_t g = nullptr;
    cudaGraphConditionalHandle h;
    int st = fasmg_check(cudaGraphCreate(&g, 0));
    if (!st) st = fasmg_check(cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault));
    if (!st) st = fasmg_check(cudaStreamBeginCaptureToGraph(E.stream, g, nullptr, nullptr, 0,
                                                             cudaStreamCaptureModeThreadLocal));
    if (st) { if (g) cudaGraphDestroy(g); return st; }
    if (E.dim == 3) capture_iteration<3>(E, ps != 0, h);
    else capture_iteration<2>(E, ps != 0, h);
    // the WHILE node after the first iteration's k_conv
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    st = fasmg_check(cudaStreamGetCaptureInfo(E.stream, &cs, nullptr, nullptr, &deps, &ndeps));
    cudaGraphNodeParams prm = {};
    prm.type = cudaGraphNodeTypeConditional;
    prm.conditional.handle = h;
    prm.conditional.type = cudaGraphCondTypeWhile;
    prm.conditional.size = 1;
    cudaGraphNode_t cond;
    if (!st) st = fasmg_check(cudaGraphAddNode(&cond, g, deps, ndeps, &prm));
    if (!st) st = fasmg_check(cudaStreamUpdateCaptureDependencies(E.stream, &cond, 1,
                                                                  cudaStreamSetCaptureDependencies));
    cudaGraph_t g2 = nullptr;
    cudaError_t e = cudaStreamEndCapture(E.stream, &g2);
    if (!st) st = fasmg_check(e);
    if (st) { cudaGraphDestroy(g); return st; }
    cudaGraph_t body = prm.conditional.phGraph_out[0];
    st = fasmg_check(cudaStreamBeginCaptureToGraph(E.stream, body, nullptr, nullptr, 0,
                                                   cudaStreamCaptureModeThreadLocal));
    if (st) { cudaGraphDestroy(g); return st; }
    if (E.dim == 3) capture_iteration<3>(E, true, h);
    else capture_iteration<2>(E, true, h);
    cudaGraph_t b2 = nullptr;
    e = cudaStreamEndCapture(E.stream, &b2);
    if ((st = fasmg_check(e))) { cudaGraphDestroy(g); return st; }
    if ((st = fasmg_check(cudaGraphInstantiate(&E.xsolve[ps], g, 0)))) { cudaGraphDestroy(g); return st; }
    E.gsolve[ps] = g;
    return 0;
}

// leave speculation: P's interior already is the state; rebuild the pads
// the speculative norm overwrote (ghosts of X_new) from it
static void spec_cancel(Engine& E) {
    if (!E.spec_pending) return;
    long cnt = 0;
    launch_pad_fill<3>(E, 0, cnt);
    E.spec_pending = false;
}

// Tensor maps of a level's blocked array as a 4D tensor (pitch, E1, E0,
// class) for TMA boxes.
static bool encode_map(CUtensorMap* m, double* base, const Lvl& L, unsigned bx, unsigned by) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
            return false;
        enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }
    cuuint64_t dims[4] = {(cuuint64_t)L.s1, (cuuint64_t)L.E[1], (cuuint64_t)L.E[0], 8};
    cuuint64_t strides[3] = {(cuuint64_t)L.s1 * 8, (cuuint64_t)L.s0 * 8, (cuuint64_t)L.cls * 8};
    cuuint32_t box[4] = {bx, by, 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, base, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2D levels: the class arrays as a 3D tensor (pitch, E0, class)
static bool encode_map2d(CUtensorMap* m, double* base, const Lvl& L, unsigned bx, unsigned by) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
            return false;
        enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }
    cuuint64_t dims[3] = {(cuuint64_t)L.s0, (cuuint64_t)L.E[0], 4};
    cuuint64_t strides[2] = {(cuuint64_t)L.s0 * 8, (cuuint64_t)L.cls * 8};
    cuuint32_t box[3] = {bx, by, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int EA>
static int tma_attr() {
    const int sm = (int)tsw::SMEM;
    cudaError_t e = cudaFuncSetAttribute(k_sweep_tma<EA, 0x96u>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_sweep_tma<EA, 0x69u>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e == cudaSuccess && EA == -1)
        e = cudaFuncSetAttribute(k_sweep_tma<-1, 0x96u, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsw::SMEM_CORR);
    if (e == cudaSuccess && EA == -1)
        e = cudaFuncSetAttribute(k_sweep_tma<-1, 0x69u, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsw::SMEM_CORR);
    if (e == cudaSuccess && EA >= 0)
        e = cudaFuncSetAttribute(k_sweep_tma<(EA < 0 ? 0 : EA), 0x96u, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsw::SMEM_ECORR);
    if (e == cudaSuccess && EA >= 0)
        e = cudaFuncSetAttribute(k_sweep_tma<(EA < 0 ? 0 : EA), 0x69u, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsw::SMEM_ECORR);
    return fasmg_check(e);
}

// TMA maps of the levels whose half-sweeps run k_sweep_tma
template <int EA>
static int tma2d_attr() {
    const int sm = (int)tsw2::SMEM;
    cudaError_t e = cudaFuncSetAttribute(k_sweep_tma2d<EA, 0x6u>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_sweep_tma2d<EA, 0x9u>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    return fasmg_check(e);
}

// The outer norm also runs the next V-cycle's first pre-smoothing half-
// sweep into P2 (k_resid_tma<2>): 3D cell-centred unsharded TMA finest
// level, the norm on the TMA march, an X plan (first two launches the two
// complementary parity groups) and no periodic face (a periodic ghost is
// written by the opposite side's thread).
static int spec_setup(Engine& E) {
    if (const char* v = getenv("FASMG_SPEC")) E.spec = atoi(v);
    if (!E.spec || E.dim != 3 || E.ea >= 0 || E.nranks > 1 || !E.tma_ok[0] || !E.resid_tma ||
        E.masks.size() < 2 || E.nl < 2)
        return 0;
    const unsigned m0 = E.masks[0];
    if (!((m0 == 0x96u || m0 == 0x69u) && E.masks[1] == (m0 ^ 0xFFu))) return 0;
    for (int a = 0; a < 3; ++a)
        if (E.bc.kind[a][0] == BC_PERIODIC || E.bc.kind[a][1] == BC_PERIODIC) return 0;
    const Lvl& L = E.L[0];
    const size_t bytes = sizeof(double) * (size_t)L.cls * 8;
    if (int st = lvl_alloc(E, 0, 5, bytes, &E.P2)) return st;
    cudaMemsetAsync(E.P2, 0, bytes, E.stream);
    if (!encode_map(&E.mapT2, E.P2, L, tsw::HX, tsw::HY)) return 0;
    cudaError_t e = cudaFuncSetAttribute(k_resid_tma<2, -1, true, 0x96u>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, E.norm_smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_resid_tma<2, -1, true, 0x69u>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, E.norm_smem);
    if (e != cudaSuccess) return fasmg_check(e);
    E.spec_ok = true;
    return 0;
}

static int tma_setup(Engine& E) {
    if (E.sweep_variant != 4) return 0;
    long min_blocks = 1L << 21;  // FASMG_TMA_MIN: smaller levels are launch-latency bound
    if (const char* v = getenv("FASMG_TMA_MIN")) min_blocks = atol(v);
    if (E.dim == 2) {
        bool any = false;
        for (int k = 0; k < E.nl; ++k) {
            const Lvl& L = E.L[k];
            if (L.B[1] < 32 || L.B[0] < 8 || L.nblk < min_blocks) continue;
            E.tma_ok[k] = encode_map2d(&E.mapT[k], E.P[k], L, tsw2::HX, tsw2::HY) &&
                          encode_map2d(&E.mapF[k], E.F[k], L, tsw2::TX, tsw2::TY);
            any = any || E.tma_ok[k];
        }
        if (!any) return 0;
        int st = 0;
        EA_DISPATCH(2, E.ea, (st = tma2d_attr<EA>()));
        return st;
    }
    if (E.dim != 3) return 0;
    bool any = false;
    for (int k = 0; k < E.nl; ++k) {
        const Lvl& L = E.L[k];
        if (L.B[2] < 32 || L.B[1] < 8 || L.nblk < min_blocks) continue;
        E.tma_ok[k] = encode_map(&E.mapT[k], E.P[k], L, tsw::HX, tsw::HY) &&
                      encode_map(&E.mapF[k], E.F[k], L, tsw::TX, tsw::TY);
        any = any || E.tma_ok[k];
    }
    if (!any) return 0;
    if (const char* v = getenv("FASMG_RESID_TMA")) E.resid_tma = atoi(v);
    if (const char* v = getenv("FASMG_CORR_FUSE")) E.corr_fuse = atoi(v);
    if (const char* v = getenv("FASMG_CORR_CHUNK")) E.corr_chunk = atoi(v);
    if (const char* v = getenv("FASMG_CHUNK_L1")) E.chunk_l1 = atoi(v);
    if (const char* v = getenv("FASMG_TAU_CHUNK")) E.tau_chunk = atoi(v);
    if (const char* v = getenv("FASMG_NORM_CHUNK")) E.norm_chunk = atoi(v);
    {
        int dev = 0, n = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
            E.num_sms = n;
    }
    // at most 3 CTAs per SM for the norm march: the EA = 1 instantiation
    // compiles to 64 registers, so 4 CTAs fit and then stall on the MIO
    // queue (ncu: mio_throttle, 553 us vs 350 us for the cell one at 3 CTAs);
    // padding the dynamic smem to 58 KB takes the EDGE_NS V-cycle 8.43 -> 8.09 ms
    E.norm_smem = std::max((int)rsw::SMEM, 58000);
    if (const char* v = getenv("FASMG_NORM_SMEM")) E.norm_smem = std::max((int)rsw::SMEM, atoi(v));
    int st = 0;
    EA_DISPATCH(3, E.ea, (st = tma_attr<EA>()));
    if (!st) EA_DISPATCH(3, E.ea, (st = fasmg_check(cudaFuncSetAttribute(
                                        k_resid_tma<0, EA>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        E.norm_smem))));
    if (!st) EA_DISPATCH(3, E.ea, (st = fasmg_check(cudaFuncSetAttribute(
                                        k_resid_tma<0, EA, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        E.norm_smem))));
    if (!st) st = fasmg_check(cudaFuncSetAttribute(k_resid_tma<1>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)rsw::SMEM));
    if (!st) st = fasmg_check(cudaFuncSetAttribute(k_resid_tma<1, -1, true>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)rsw::SMEM));
    if (!st) st = spec_setup(E);
    if (const char* v = getenv("FASMG_EDGE_TAU")) E.edge_tau = atoi(v);
    if (const char* v = getenv("FASMG_RESID_PF")) E.resid_pf = atoi(v);
    if (const char* v = getenv("FASMG_ETAU_CHUNK")) E.etau_chunk = std::max(1, atoi(v));
    if (!st && E.ea >= 0)
        EA_DISPATCH(3, E.ea, (st = fasmg_check(cudaFuncSetAttribute(
                                  k_tau_edge_tma<(EA < 0 ? 0 : EA)>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)esw::SMEM))));
    return st;
}


// Levels from coarse_k0 down run in k_coarse_cycle: cell-centered, not
// sharded, at most coarse_max blocks.
static int coarse_setup(Engine& E) {
    if (const char* v = getenv("FASMG_COARSE_MAX")) E.coarse_max = atol(v);
    if (const char* v = getenv("FASMG_COARSE_CS")) E.coarse_cs = std::max(1, std::min(16, atoi(v)));
    // Slab engines run it on their replicated coarse levels (k0 >= kg: no
    // exchange inside).  (Round 1 kept slab engines off it after 8 virtual
    // ranks at 512^3 hung; the cause was lazy module loading during a capture
    // -- fixed by fasmg_engine_prepare -- not the cluster launch.)
    // Edge fields keep per-level launches: the same scheme with the edge
    // transfers' phases (residual, pads, two restrictions, pad fill, pinit,
    // correction, prolongation; all bitwise) measured SLOWER than the
    // launches it replaced (EDGE_NS 512^3 V-cycle 8.26 -> 8.41 ms: ~16
    // cluster-barrier phases per level against ~2.5 us per graph launch).
    if (E.ea >= 0 || E.coarse_max <= 0 || E.masks.size() > 16) return 0;
    int k0 = E.nl;
    while (k0 > 0 && !E.sharded(k0 - 1) && E.L[k0 - 1].nblk <= E.coarse_max) --k0;
    if (k0 >= E.nl) return 0;
    CoarseArgs h;
    memset(&h, 0, sizeof(h));
    for (int k = 0; k < E.nl; ++k) {
        h.P[k] = E.P[k];
        h.F[k] = E.F[k];
        h.L[k] = E.L[k];
    }
    h.bc = E.bc;
    h.k0 = k0;
    int k1 = E.nl - 1;  // first level small enough for one CTA (<= ~2 blocks per thread)
    while (k1 > k0 && E.L[k1 - 1].nblk <= 1024) --k1;
    h.k1 = k1;
    h.nl = E.nl;
    h.s = E.s;
    h.nm = (int)E.masks.size();
    for (int j = 0; j < h.nm; ++j) h.masks[j] = E.masks[j];
    int st = fasmg_check(cudaMalloc(&E.dcoarse, sizeof(CoarseArgs)));
    if (!st) st = fasmg_check(cudaMemcpy(E.dcoarse, &h, sizeof(h), cudaMemcpyHostToDevice));
    if (!st && E.coarse_cs > 8) {
        st = fasmg_check(cudaFuncSetAttribute(E.dim == 3 ? (const void*)k_coarse_cycle<3>
                                                         : (const void*)k_coarse_cycle<2>,
                                              cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    }
    if (!st) E.coarse_k0 = k0;
    return st;
}

static Lvl make_lvl(int dim, const int* n, int ea, double dmin, double dmax, double a,
                    double b) {
    Lvl L;
    memset(&L, 0, sizeof(L));
    L.dim = dim;
    L.ea = ea;
    L.nblk = 1;
    for (int t = 0; t < 3; ++t) {
        L.n[t] = t < dim ? n[t] : 2;
        L.B[t] = L.n[t] / 2;
        L.E[t] = L.B[t] + 2;
        if (t < dim) L.nblk *= L.B[t];
    }
    int last = dim - 1;
    long pitch = ((long)L.E[last] + OFF + 3) / 4 * 4;
    if (dim == 3) {
        L.s1 = pitch;
        L.s0 = pitch * L.E[1];
        L.cls = L.s0 * L.E[0];
    } else {
        L.s1 = 1;
        L.s0 = pitch;
        L.cls = pitch * L.E[0];
    }
    L.cls = (L.cls + 31) / 32 * 32;  // 256-byte aligned class arrays
    L.off0 = 0;
    L.G0 = L.B[0];
    // scalars exactly as the reference computes them (PKG/grid.py:71-73,
    // PKG/smoothers.py:143-144, PKG/stencil.py:37-38,58)
    L.h = (dmax - dmin) / n[0];
    L.h2 = L.h * L.h;
    L.inv_h2 = 1.0 / (L.h * L.h);
    L.a = a;
    L.b = b;
    L.denom = a * L.h2 + (double)(2 * dim) * b;
    L.rden = 1.0 / L.denom;
    return L;
}

}  // namespace fasmg

using namespace fasmg;

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

// masks: one uint32 per color group (classes updated after one ghost
// refresh); the smoother of one smoothing step runs them in order.
// Create an engine.  nranks > 1: this engine owns the axis-0 slab `rank` of
// every level whose block-plane count divides evenly into >= min_planes
// (even) planes per rank; coarser levels are replicated on every rank.  Peer
// pointers are supplied later by fasmg_engine_connect.
void* fasmg_engine_create_slab(int dim, const int* n, int ea, double dmin, double dmax,
                               int mesh_level, double a, double b, const int* kinds,
                               const double* vals, int nmasks, const unsigned* masks, int s,
                               void* stream, int nranks, int rank, int min_planes) {
    if (dim != 2 && dim != 3) { fasmg_set_error(FASMG_EINVAL, "dim must be 2 or 3"); return nullptr; }
    if (mesh_level < 1 || mesh_level > 30) { fasmg_set_error(FASMG_EINVAL, "bad mesh_level"); return nullptr; }
    for (int t = 0; t < dim; ++t)
        if (n[t] % (1 << mesh_level) != 0 || (n[t] >> mesh_level) % 2 != 0) {
            fasmg_set_error(FASMG_EINVAL, "grid does not stay even through mesh_level coarsenings");
            return nullptr;
        }
    // launch geometries put (block) extents of the outer axes on gridDim.y/z
    // (pack_grid, face_grid), which CUDA caps at 65535
    if ((dim == 3 && (n[0] + 2 > 65535 || n[1] + 2 > 2 * 65535)) ||
        (dim == 2 && n[0] + 2 > 2 * 65535)) {
        fasmg_set_error(FASMG_EINVAL, "grid extent exceeds the 65535 CUDA grid-dimension limit");
        return nullptr;
    }
    if (nranks < 1 || rank < 0 || rank >= nranks) {
        fasmg_set_error(FASMG_EINVAL, "bad nranks/rank");
        return nullptr;
    }
    if (nranks > 1 && kinds[0] == BC_PERIODIC) {
        fasmg_set_error(FASMG_EINVAL, "slab decomposition needs a non-periodic axis 0");
        return nullptr;
    }
    Engine* E = new Engine();
    E->dim = dim;
    E->ea = ea;
    E->nl = mesh_level + 1;
    E->s = s;
    E->stream = (cudaStream_t)stream;
    E->nranks = nranks;
    if (t_arena && nranks == 1) {  // slab engines export their arrays: never shared
        E->arena = t_arena;
        ++t_arena->refs;
    }
    E->rank = rank;
    for (int t = 0; t < 3; ++t)
        for (int sd = 0; sd < 2; ++sd) {
            E->bc.kind[t][sd] = t < dim ? kinds[2 * t + sd] : 0;
            E->bc.val[t][sd] = t < dim ? vals[2 * t + sd] : 0.0;
            E->bch.kind[t][sd] = E->bc.kind[t][sd];
            E->bch.val[t][sd] = 0.0;  // PKG/boundary.py:83-87
        }
    for (int t = 0; t < nmasks; ++t)
        if (!mask_supported(dim, masks[t])) {
            fasmg_set_error(FASMG_EINVAL, "unsupported class mask in smoothing plan");
            delete E;
            return nullptr;
        }
    E->masks.assign(masks, masks + nmasks);
    if (const char* v = getenv("FASMG_SWEEP_VARIANT")) E->sweep_variant = atoi(v);
    if (const char* v = getenv("FASMG_MARCH_CHUNK")) E->march_chunk = std::max(0, atoi(v));
    if (const char* v = getenv("FASMG_TILE_Y")) g_tile_y = std::max(1, atoi(v));
    if (const char* v = getenv("FASMG_SWEEP_MINB")) E->sweep_minb = atoi(v);
    if (const char* v = getenv("FASMG_EDGE_FAST")) E->edge_fast = atoi(v);
    if (const char* v = getenv("FASMG_FUSE_PUSH")) E->fuse_push = atoi(v);
    if (nranks > 1) E->edge_fast = 1;  // the slab-aware edge transfers
    // sharded levels: a prefix of the hierarchy, never the coarsest
    E->kg = 0;
    if (nranks > 1) {
        const int mp = std::max(2, min_planes);
        for (int k = 0; k < E->nl - 1; ++k) {
            const int B0 = (n[0] >> k) / 2;
            if (B0 % nranks || (B0 / nranks) % 2 || B0 / nranks < mp) break;
            E->kg = k + 1;
        }
        if (E->kg == 0) {
            fasmg_set_error(FASMG_EINVAL, "grid too small to split into slabs");
            delete E;
            return nullptr;
        }
    }
    int nn[3] = {n[0], n[1], dim == 3 ? n[2] : 2};
    for (int k = 0; k < E->nl; ++k) {
        Lvl L = make_lvl(dim, nn, ea, dmin, dmax, a, b);
        if (E->sharded(k)) {  // local slab: nb planes + the two halo/pad planes
            const int nbp = L.B[0] / nranks;
            L.off0 = rank * nbp;
            L.G0 = L.B[0];
            L.B[0] = nbp;
            L.E[0] = nbp + 2;
            L.nblk = (long)nbp * L.B[1] * (dim == 3 ? L.B[2] : 1);
            L.cls = (L.s0 * L.E[0] + 31) / 32 * 32;
        }
        E->L[k] = L;
        size_t bytes = sizeof(double) * (size_t)E->L[k].cls * (1u << dim);
        if (lvl_alloc(*E, k, 0, bytes, &E->P[k]) || lvl_alloc(*E, k, 1, bytes, &E->F[k])) {
            delete E;
            return nullptr;
        }
        cudaMemsetAsync(E->P[k], 0, bytes, E->stream);
        cudaMemsetAsync(E->F[k], 0, bytes, E->stream);
        if (ea < 0 && dim == 3 && nranks == 1 && k >= 1) {  // pinit for the fused correction
            if (lvl_alloc(*E, k, 2, bytes, &E->PI[k])) { delete E; return nullptr; }
            cudaMemsetAsync(E->PI[k], 0, bytes, E->stream);
        }
        if (ea >= 0) {
            // R[0] (the finest residual of the unfused edge tau pass) is
            // allocated after tma_setup, only if that pass is needed
            if (k >= 1 && lvl_alloc(*E, k, 2, bytes, &E->R[k])) { delete E; return nullptr; }
            if (k >= 1 && lvl_alloc(*E, k, 3, bytes, &E->PI[k])) { delete E; return nullptr; }
            if (k >= 1) cudaMemsetAsync(E->R[k], 0, bytes, E->stream);
            if (k >= 1) cudaMemsetAsync(E->PI[k], 0, bytes, E->stream);
        }
        for (int t = 0; t < dim; ++t) nn[t] /= 2;
    }
    E->npart = (int)tile_ctas(tile_of(E->L[0]));
    if (int st = coarse_setup(*E)) { delete E; fasmg_set_error(st, "engine setup (coarse cluster) failed"); return nullptr; }
    if (int st = tma_setup(*E)) { delete E; fasmg_set_error(st, "engine setup (TMA maps) failed"); return nullptr; }
    if (ea >= 0 && !(dim == 3 && edge_tau_level(*E, 0))) {  // the unfused finest tau pass
        const size_t bytes = sizeof(double) * (size_t)E->L[0].cls * (1u << dim);
        if (lvl_alloc(*E, 0, 2, bytes, &E->R[0])) { delete E; return nullptr; }
        cudaMemsetAsync(E->R[0], 0, bytes, E->stream);
    }
    if (fasmg_check(cudaMalloc(&E->part, sizeof(double) * E->npart)) ||
        fasmg_check(cudaMalloc(&E->dsum, sizeof(double))) ||
        fasmg_check(cudaMallocHost(&E->hsum, sizeof(double))) ||
        fasmg_check(cudaMalloc(&E->flags, sizeof(long long) * nranks)) ||
        fasmg_check(cudaMalloc(&E->cnt, sizeof(long long) * 2 * nranks)) ||
        fasmg_check(cudaMalloc(&E->allpart, sizeof(double) * nranks))) {
        delete E;
        return nullptr;
    }
    cudaMemsetAsync(E->flags, 0, sizeof(long long) * nranks, E->stream);
    cudaMemsetAsync(E->cnt, 0, sizeof(long long) * 2 * nranks, E->stream);
    cudaMemsetAsync(E->allpart, 0, sizeof(double) * nranks, E->stream);
    if (nranks == 1) {
        Engine::Peer me;
        for (int k = 0; k < 32; ++k) { me.P[k] = E->P[k]; me.F[k] = E->F[k]; }
        me.flags = E->flags;
        me.allpart = E->allpart;
        E->peers.assign(1, me);
    }
    if (fasmg_check(cudaStreamSynchronize(E->stream))) { delete E; return nullptr; }
    return E;
}

void* fasmg_engine_create(int dim, const int* n, int ea, double dmin, double dmax,
                          int mesh_level, double a, double b, const int* kinds,
                          const double* vals, int nmasks, const unsigned* masks, int s,
                          void* stream) {
    return fasmg_engine_create_slab(dim, n, ea, dmin, dmax, mesh_level, a, b, kinds, vals,
                                    nmasks, masks, s, stream, 1, 0, 0);
}

void* fasmg_arena_create(void) { return new Arena(); }

void fasmg_arena_release(void* h) {
    Arena* A = (Arena*)h;
    if (!A || --A->refs > 0) return;
    for (auto& kv : A->buf)
        if (kv.second.second) cudaFree(kv.second.second);
    delete A;
}

// fasmg_engine_create with the level arrays taken from `arena` (shared with
// the other engines created in it; they must not run concurrently)
void* fasmg_engine_create_in(int dim, const int* n, int ea, double dmin, double dmax,
                             int mesh_level, double a, double b, const int* kinds,
                             const double* vals, int nmasks, const unsigned* masks, int s,
                             void* stream, void* arena) {
    t_arena = (Arena*)arena;
    void* h = fasmg_engine_create_slab(dim, n, ea, dmin, dmax, mesh_level, a, b, kinds, vals,
                                       nmasks, masks, s, stream, 1, 0, 0);
    t_arena = nullptr;
    return h;
}

// Number of device pointers fasmg_engine_export writes: P[0..nl), F[0..nl),
// flags, allpart.
int fasmg_engine_export_count(void* h) { return 3 * ((Engine*)h)->nl + 2; }

int fasmg_engine_export(void* h, unsigned long long* out) {
    Engine* E = (Engine*)h;
    int t = 0;
    for (int k = 0; k < E->nl; ++k) out[t++] = (unsigned long long)E->P[k];
    for (int k = 0; k < E->nl; ++k) out[t++] = (unsigned long long)E->F[k];
    for (int k = 0; k < E->nl; ++k) out[t++] = (unsigned long long)E->R[k];
    out[t++] = (unsigned long long)E->flags;
    out[t++] = (unsigned long long)E->allpart;
    return 0;
}

// all: nranks consecutive export arrays, pointers valid in THIS process
// (the peer's own pointers for virtual ranks on one device; CUDA-IPC
// mappings for one process per GPU)
int fasmg_engine_connect(void* h, const unsigned long long* all, int nranks) {
    Engine* E = (Engine*)h;
    if (nranks != E->nranks) return fasmg_set_error(FASMG_EINVAL, "nranks mismatch");
    const int per = 3 * E->nl + 2;
    E->peers.assign(nranks, Engine::Peer());
    for (int r = 0; r < nranks; ++r) {
        const unsigned long long* x = all + (long)r * per;
        Engine::Peer& pr = E->peers[r];
        for (int k = 0; k < 32; ++k) pr.P[k] = pr.F[k] = pr.R[k] = nullptr;
        for (int k = 0; k < E->nl; ++k) {
            pr.P[k] = (double*)x[k];
            pr.F[k] = (double*)x[E->nl + k];
            pr.R[k] = (double*)x[2 * E->nl + k];
        }
        pr.flags = (long long*)x[3 * E->nl];
        pr.allpart = (double*)x[3 * E->nl + 1];
    }
    return 0;
}

// [kg, local planes of level 0, global offset of level 0]
int fasmg_engine_slab_info(void* h, int* out) {
    Engine* E = (Engine*)h;
    out[0] = E->kg;
    out[1] = E->L[0].B[0];
    out[2] = E->L[0].off0;
    return 0;
}

// full halo exchange of level 0 (after loading a slab)
int fasmg_engine_sync_halos(void* h) {
    Engine* E = (Engine*)h;
    long cnt = 0;
    if (E->dim == 3) halo_exchange<3>(*E, 0, 0xFFu, cnt);
    else halo_exchange<2>(*E, 0, 0xFu, cnt);
    return fasmg_check_launch();
}

int fasmg_ipc_get_handle(void* ptr, unsigned char* out64) {
    cudaIpcMemHandle_t hd;
    int st = fasmg_check(cudaIpcGetMemHandle(&hd, ptr));
    if (!st) memcpy(out64, &hd, sizeof(hd));
    return st;
}

int fasmg_ipc_open_handle(const unsigned char* in64, void** ptr) {
    cudaIpcMemHandle_t hd;
    memcpy(&hd, in64, sizeof(hd));
    return fasmg_check(cudaIpcOpenMemHandle(ptr, hd, cudaIpcMemLazyEnablePeerAccess));
}

int fasmg_ipc_close_handle(void* ptr) { return fasmg_check(cudaIpcCloseMemHandle(ptr)); }

void fasmg_engine_destroy(void* h) {
    Engine* E = (Engine*)h;
    if (!E) return;
    cudaStreamSynchronize(E->stream);
    for (int a = 0; a < 2; ++a) {
        for (int b = 0; b < 2; ++b) {
            if (E->execs[a][b]) cudaGraphExecDestroy(E->execs[a][b]);
            if (E->graphs[a][b]) cudaGraphDestroy(E->graphs[a][b]);
        }
        if (E->xsolve[a]) cudaGraphExecDestroy(E->xsolve[a]);
        if (E->gsolve[a]) cudaGraphDestroy(E->gsolve[a]);
    }
    if (E->dhist) cudaFree(E->dhist);
    if (E->dit) cudaFree(E->dit);
    if (E->dctl) cudaFree(E->dctl);
    if (E->hbuf) cudaFreeHost(E->hbuf);
    for (void* ptr : E->owned) cudaFree(ptr);
    if (E->arena) {
        if (E->arena->last == E) E->arena->last = nullptr;
        fasmg_arena_release(E->arena);
    }
    cudaFree(E->part);
    cudaFree(E->dsum);
    cudaFreeHost(E->hsum);
    cudaFree(E->flags);
    cudaFree(E->cnt);
    cudaFree(E->allpart);
    if (E->dcoarse) cudaFree(E->dcoarse);
    delete E;
}

// Load p and f (natural core views) into the engine's finest level.
int fasmg_engine_load(void* h, const double* pcore, const long* ps, const double* fcore,
                      const long* fs) {
    Engine* E = (Engine*)h;
    E->spec_pending = false;  // new state: P2 no longer describes it
    if (E->arena && E->arena->last != E) {  // another engine used the arrays: start fresh
        // (the finest P and F are skipped: the pack below writes their whole
        // core box, pads included, before anything reads them)
        for (int k = 0; k < E->nl; ++k) {
            const size_t bytes = sizeof(double) * (size_t)E->L[k].cls * (1u << E->dim);
            for (double* q : {E->P[k], E->F[k], E->R[k], E->PI[k]})
                if (q && !(k == 0 && (q == E->P[0] || q == E->F[0])))
                    cudaMemsetAsync(q, 0, bytes, E->stream);
        }
        E->arena->last = E;
    }
    const Lvl& L = E->L[0];
    int e[3];
    for (int a = 0; a < 3; ++a) e[a] = a < E->dim ? (a == E->ea ? L.n[a] + 1 : L.n[a] + 2) : 1;
    if (E->sharded(0)) {  // rank-local slab (+1 ghost plane each side)
        e[0] = 2 * L.B[0] + 2;
        if (E->ea == 0 && E->rank == E->nranks - 1) e[0] -= 1;  // edge axis ends at the wall n
    }
    dim3 pg, pb;
    pack_grid(E->dim, e[0], e[1], e[2], pg, pb);
    if (E->dim == 3) {
        k_pack<3><<<pg, pb, 0, E->stream>>>(pcore, ps[0], ps[1], ps[2], E->P[0], L, e[0], e[1],
                                            e[2]);
        k_pack<3><<<pg, pb, 0, E->stream>>>(fcore, fs[0], fs[1], fs[2], E->F[0], L, e[0], e[1],
                                            e[2]);
    } else {
        k_pack<2><<<pg, pb, 0, E->stream>>>(pcore, ps[0], ps[1], 0, E->P[0], L, e[0], e[1], 1);
        k_pack<2><<<pg, pb, 0, E->stream>>>(fcore, fs[0], fs[1], 0, E->F[0], L, e[0], e[1], 1);
    }
    long cnt = 0;
    if (E->dim == 3) launch_pad_fill<3>(*E, 0, cnt);
    else launch_pad_fill<2>(*E, 0, cnt);
    return fasmg_check_launch();
}

// Store the finest-level solution interior into a natural core view.
int fasmg_engine_store(void* h, double* pcore, const long* ps) {
    Engine* E = (Engine*)h;
    const Lvl& L = E->L[0];
    int m[3];
    for (int a = 0; a < 3; ++a) m[a] = a < E->dim ? (a == E->ea ? L.n[a] - 1 : L.n[a]) : 1;
    if (E->sharded(0)) {
        m[0] = 2 * L.B[0];
        if (E->ea == 0 && E->rank == E->nranks - 1) m[0] -= 1;  // the last node is the wall
    }
    dim3 pg, pb;
    pack_grid(E->dim, m[0], m[1], m[2], pg, pb);
    if (E->dim == 3)
        k_unpack<3><<<pg, pb, 0, E->stream>>>(E->P[0], L, pcore, ps[0], ps[1], ps[2], m[0], m[1],
                                              m[2]);
    else
        k_unpack<2><<<pg, pb, 0, E->stream>>>(E->P[0], L, pcore, ps[0], ps[1], 0, m[0], m[1], 1);
    return fasmg_check_launch();
}

// Enqueue `count` V-cycles; when with_norm, each is followed by the outer
// residual norm's sum of squares, and the LAST one is copied to *sumsq
// after synchronizing (returned through the pinned scalar).
int fasmg_engine_run(void* h, int count, int with_norm, double* sumsq, int use_graph) {
    Engine* E = (Engine*)h;
    int st;
    for (int it = 0; it < count; ++it) {
        if (use_graph) {
            cudaGraphExec_t* ex;
            cudaGraph_t* g;
            graph_slot(*E, with_norm != 0, &g, &ex);
            if (!*ex && (st = capture(*E, with_norm != 0, g, ex))) return st;
            if ((st = fasmg_check(cudaGraphLaunch(*ex, E->stream)))) return st;
        } else {
            long cnt = 0;
            E->cap_pending = E->spec_ok && E->spec_pending;
            E->cap_spec = E->spec_ok && with_norm;
            if (E->dim == 3) {
                launch_vcycle<3>(*E, cnt);
                if (with_norm) launch_norm<3>(*E, cnt);
            } else {
                launch_vcycle<2>(*E, cnt);
                if (with_norm) launch_norm<2>(*E, cnt);
            }
            E->cap_pending = E->cap_spec = false;
            if (with_norm)
                cudaMemcpyAsync(E->hsum, E->dsum, sizeof(double), cudaMemcpyDeviceToHost,
                                E->stream);
            if ((st = fasmg_check_launch())) return st;
        }
        after_launch(*E, with_norm != 0);
    }
    if (with_norm) {
        if ((st = fasmg_check(cudaStreamSynchronize(E->stream)))) return st;
        *sumsq = *E->hsum;
    }
    return 0;
}

// Asynchronous variant for ranks that must run concurrently (virtual ranks
// on one device, whose graphs wait on each other): enqueue `count` V-cycles
// (+ norm) and return; fasmg_engine_result waits and reads the last sum.
int fasmg_engine_launch(void* h, int count, int with_norm) {
    Engine* E = (Engine*)h;
    int st;
    for (int it = 0; it < count; ++it) {
        cudaGraphExec_t* ex;
        cudaGraph_t* g;
        graph_slot(*E, with_norm != 0, &g, &ex);
        if (!*ex && (st = capture(*E, with_norm != 0, g, ex))) return st;
        if ((st = fasmg_check(cudaGraphLaunch(*ex, E->stream)))) return st;
        after_launch(*E, with_norm != 0);
    }
    return 0;
}

// Capture and instantiate the V-cycle graph (with_norm selects the variant)
// without launching it.  Ranks that share a device must all be prepared
// before any of them launches: capturing a kernel for the first time loads
// its module lazily (CUDA_MODULE_LOADING=LAZY, the default), and a lazy
// load waits for the device's running kernels -- which include the peers'
// k_wait spins on this rank, so launching one rank while another is still
// capturing deadlocks until k_wait's guard traps.
int fasmg_engine_prepare(void* h, int with_norm) {
    Engine* E = (Engine*)h;
    cudaGraphExec_t* ex;
    cudaGraph_t* g;
    graph_slot(*E, with_norm != 0, &g, &ex);
    if (!*ex) return capture(*E, with_norm != 0, g, ex);
    return 0;
}

// A whole outer solve loop (PKG/fas.py:147-154) as one graph launch: up to
// k_max V-cycles + norms on the loaded state, stopping on the device at the
// first res = scale*sqrt(sumsq) <= tol.  history: host array of k_max doubles;
// *iters = V-cycles run.  Slab ranks: every rank's norm is the same
// rank-ordered sum, so the ranks stop together.
//
// the device loop's buffers (each on its own: a failed allocation is
// retried by the next call) and its graph for the current speculation state
static int solve_prepare(Engine& E) {
    int st;
    if (!E.dhist && (st = fasmg_check(cudaMalloc(&E.dhist, sizeof(double) * SOLVE_CAP)))) return st;
    if (!E.dit && (st = fasmg_check(cudaMalloc(&E.dit, sizeof(int))))) return st;
    if (!E.dctl && (st = fasmg_check(cudaMalloc(&E.dctl, sizeof(double) * 3)))) return st;
    if (!E.hbuf && (st = fasmg_check(cudaMallocHost(&E.hbuf, sizeof(double) * (SOLVE_CAP + 4)))))
        return st;
    const int ps = E.spec_ok && E.spec_pending ? 1 : 0;
    if (!E.xsolve[ps] && (st = build_solve_graph(E, ps))) return st;
    return 0;
}

// Capture the device loop's graph before any rank launches (slab ranks on
// one device: a capture that lazily loads a module waits for running
// kernels, i.e. for peers spinning on this rank -- see fasmg_engine_prepare).
int fasmg_engine_prepare_solve(void* h) { return solve_prepare(*(Engine*)h); }

// Enqueue the device loop (no host synchronization): slab ranks enqueue on
// every rank first, then wait.  Every rank's norm is the same rank-ordered
// sum (launch_norm), so all ranks take the same decisions in lockstep.
int fasmg_engine_solve_launch(void* h, int k_max, double tol, double scale) {
    Engine* E = (Engine*)h;
    if (k_max < 1 || k_max > SOLVE_CAP) return fasmg_set_error(FASMG_EINVAL, "k_max out of range");
    int st;
    if ((st = solve_prepare(*E))) return st;
    const int ps = E->spec_ok && E->spec_pending ? 1 : 0;
    E->hbuf[0] = tol;
    E->hbuf[1] = scale;
    E->hbuf[2] = (double)k_max;
    if ((st = fasmg_check(cudaMemcpyAsync(E->dctl, E->hbuf, sizeof(double) * 3,
                                          cudaMemcpyHostToDevice, E->stream)))) return st;
    if ((st = fasmg_check(cudaMemsetAsync(E->dit, 0, sizeof(int), E->stream)))) return st;
    if ((st = fasmg_check(cudaGraphLaunch(E->xsolve[ps], E->stream)))) return st;
    int* hcount = (int*)(E->hbuf + SOLVE_CAP + 3);
    if ((st = fasmg_check(cudaMemcpyAsync(hcount, E->dit, sizeof(int), cudaMemcpyDeviceToHost,
                                          E->stream)))) return st;
    if ((st = fasmg_check(cudaMemcpyAsync(E->hbuf + 3, E->dhist, sizeof(double) * k_max,
                                          cudaMemcpyDeviceToHost, E->stream)))) return st;
    E->spec_pending = E->spec_ok;  // every iteration ends with the fused norm
    return 0;
}

// Wait for the loop fasmg_engine_solve_launch enqueued; its history (host,
// up to k_max doubles) and iteration count.
int fasmg_engine_solve_wait(void* h, double* history, int* iters) {
    Engine* E = (Engine*)h;
    if (!E->hbuf) return fasmg_set_error(FASMG_EINVAL, "no device solve loop was launched");
    int st;
    if ((st = fasmg_check(cudaStreamSynchronize(E->stream)))) return st;
    const int n = *(const int*)(E->hbuf + SOLVE_CAP + 3);
    *iters = n;
    for (int i = 0; i < n; ++i) history[i] = E->hbuf[3 + i];
    return 0;
}

int fasmg_engine_solve(void* h, int k_max, double tol, double scale, double* history,
                       int* iters) {
    int st = fasmg_engine_solve_launch(h, k_max, tol, scale);
    return st ? st : fasmg_engine_solve_wait(h, history, iters);
}

int fasmg_engine_result(void* h, double* sumsq) {
    Engine* E = (Engine*)h;
    int st = fasmg_check(cudaStreamSynchronize(E->stream));
    if (!st) *sumsq = *E->hsum;
    return st;
}

// Debug/test access to a level's blocked arrays: geometry
// [cls, s0, s1, E0, E1, E2, B0(local), off0, G0] and a raw device copy.
int fasmg_engine_level_geom(void* h, int k, long* out) {
    Engine* E = (Engine*)h;
    if (k < 0 || k >= E->nl) return fasmg_set_error(FASMG_EINVAL, "level out of range");
    const Lvl& L = E->L[k];
    long v[9] = {L.cls, L.s0, L.s1, L.E[0], L.E[1], L.E[2], L.B[0], L.off0, L.G0};
    for (int t = 0; t < 9; ++t) out[t] = v[t];
    return 0;
}

int fasmg_engine_level_copy(void* h, int k, int which, double* dst) {
    Engine* E = (Engine*)h;
    spec_cancel(*E);
    if (k < 0 || k >= E->nl) return fasmg_set_error(FASMG_EINVAL, "level out of range");
    const double* src = which == 0 ? E->P[k] : (which == 1 ? E->F[k] : nullptr);
    if (!src) return fasmg_set_error(FASMG_EINVAL, "no such array");
    int st = fasmg_check(cudaStreamSynchronize(E->stream));
    if (st) return st;
    return fasmg_check(cudaMemcpy(dst, src, sizeof(double) * E->L[k].cls * (1u << E->dim),
                                  cudaMemcpyDeviceToDevice));
}

// Residual sum of squares of the current finest state (no V-cycle).
int fasmg_engine_residual_sumsq(void* h, double* sumsq) {
    Engine* E = (Engine*)h;
    spec_cancel(*E);
    long cnt = 0;
    if (E->dim == 3) launch_norm<3>(*E, cnt);
    else launch_norm<2>(*E, cnt);
    cudaMemcpyAsync(E->hsum, E->dsum, sizeof(double), cudaMemcpyDeviceToHost, E->stream);
    int st = fasmg_check(cudaStreamSynchronize(E->stream));
    if (!st) *sumsq = *E->hsum;
    return st;
}

// Time `reps` smoothing half-sweep launches of level k (the smoother's
// masks in order, cycling) with CUDA events on the engine stream; returns
// the mean duration of one launch in *ms.  This is the live per-launch
// timing bench.py reports for the roofline.
int fasmg_engine_time_sweeps(void* h, int k, int reps, double* ms) {
    Engine* E = (Engine*)h;
    spec_cancel(*E);
    if (k < 0 || k >= E->nl || reps < 1) return fasmg_set_error(FASMG_EINVAL, "bad level/reps");
    cudaEvent_t a, b;
    int st = fasmg_check(cudaEventCreate(&a));
    if (st) return st;
    if ((st = fasmg_check(cudaEventCreate(&b)))) { cudaEventDestroy(a); return st; }
    const Tile t = tile_of(E->L[k]);
    cudaEventRecord(a, E->stream);
    for (int r = 0; r < reps; ++r) {
        unsigned m = E->masks[r % E->masks.size()];
        if (E->dim == 3) EA_DISPATCH(3, E->ea, (sweep_mask<3, EA>(*E, k, m, t)));
        else EA_DISPATCH(2, E->ea, (sweep_mask<2, EA>(*E, k, m, t)));
    }
    cudaEventRecord(b, E->stream);
    st = fasmg_check(cudaEventSynchronize(b));
    float f = 0.f;
    if (!st) st = fasmg_check(cudaEventElapsedTime(&f, a, b));
    *ms = f / reps;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return st ? st : fasmg_check_launch();
}

// kernels launched per V-cycle (with_norm: V-cycle + outer residual norm),
// counted while building the graph; 0 before the first captured run
long fasmg_engine_kernels_per_vcycle(void* h, int with_norm) {
    Engine* E = (Engine*)h;
    // with_norm 2: one iteration of the device solve loop (fasmg_engine_solve)
    if (with_norm == 2) return E->kernels_per_solve_iter;
    return with_norm ? E->kernels_per_vcycle_norm : E->kernels_per_vcycle;
}

// Device pointer and geometry of a level's blocked arrays (tests/bench).
int fasmg_engine_level_info(void* h, int k, long* info) {
    Engine* E = (Engine*)h;
    if (k < 0 || k >= E->nl) return fasmg_set_error(FASMG_EINVAL, "level out of range");
    const Lvl& L = E->L[k];
    info[0] = L.nblk;
    info[1] = L.cls;
    info[2] = L.n[0];
    info[3] = L.n[1];
    info[4] = L.n[2];
    return 0;
}

}  // extern "C"
