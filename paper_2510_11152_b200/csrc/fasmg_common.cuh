// fasmg_common.cuh -- shared device helpers for the B200 FAS multigrid path.
//
// Arithmetic contract: every expression follows the reference association
// order (KER/numpy_backend.py, cited per kernel), with explicit
// __dadd_rn/__dmul_rn/__dsub_rn/__ddiv_rn so that no FMA contraction can
// occur regardless of compiler flags (the build also passes -fmad=false).
// That makes every per-point value bitwise identical to the reference CPU
// path, which the residual-history parity
// requires.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fasmg {

// Thread -> points of an e0 x e1 (x e2) box without 64-bit integer division:
// a CTA covers BOX_X points of the innermost axis x BOX_Y rows of the next
// one, and (3D) every thread walks BOX_Z consecutive points of the outermost
// axis, so a 512^3 box is 131K CTAs of 256 threads instead of 1M CTAs of
// 128 (the one-point-per-thread mapping was CTA-launch-bound: k_div ran at
// 1.9 TB/s).  Launch with box_grid / box_block and loop z < box_zn(dim).
constexpr int BOX_X = 128, BOX_Y = 2, BOX_Z = 4;
__host__ __device__ __forceinline__ int box_zn(int dim) { return dim == 3 ? BOX_Z : 1; }
__device__ __forceinline__ bool box_coords(int dim, int e0, int e1, int e2, int z, int* x) {
    if (dim == 3) {
        x[2] = blockIdx.x * blockDim.x + threadIdx.x;
        x[1] = blockIdx.y * blockDim.y + threadIdx.y;
        x[0] = blockIdx.z * BOX_Z + z;
        return x[2] < e2 && x[1] < e1 && x[0] < e0;
    }
    x[1] = blockIdx.x * blockDim.x + threadIdx.x;
    x[0] = blockIdx.y * blockDim.y + threadIdx.y;
    x[2] = 0;
    return x[1] < e1 && x[0] < e0;
}
// gridDim.y / gridDim.z are capped at 65535: callers reject larger boxes
// with FASMG_EINVAL up front.
static inline bool box_fits(int dim, int e0, int e1) {
    return dim == 3 ? ((e0 + BOX_Z - 1) / BOX_Z <= 65535 && (e1 + BOX_Y - 1) / BOX_Y <= 65535)
                    : (e0 + BOX_Y - 1) / BOX_Y <= 65535;
}
static inline dim3 box_grid(int dim, int e0, int e1, int e2) {
    if (dim == 3)
        return dim3((unsigned)((e2 + BOX_X - 1) / BOX_X), (unsigned)((e1 + BOX_Y - 1) / BOX_Y),
                    (unsigned)((e0 + BOX_Z - 1) / BOX_Z));
    return dim3((unsigned)((e1 + BOX_X - 1) / BOX_X), (unsigned)((e0 + BOX_Y - 1) / BOX_Y), 1u);
}
static inline dim3 box_block() { return dim3(BOX_X, BOX_Y, 1); }


// ---------------------------------------------------------------------------
// exact fp64 primitives (no contraction)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double ad(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sb(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ml(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dv(double a, double b) { return __ddiv_rn(a, b); }
// a / d correctly rounded (bitwise __ddiv_rn) from r = RN(1/d), computed
// once on the host by IEEE division: q0 = RN(a*r) is within 1.5 ulp of a/d,
// one fma-Newton correction brings q1 within 1 ulp, and Markstein's theorem
// (r within 1/2 ulp of 1/d, q1 within 1 ulp of a/d, remainder exact by fma)
// makes q2 = RN(q1 + (a - d*q1)*r) the correctly rounded quotient.  Valid for
// normal (non-subnormal, finite) quotients; a zero numerator keeps its sign.
// 5 fp64 instructions instead of __ddiv_rn's reciprocal iteration and
// slow-path branch (verified against __ddiv_rn by fasmg_selftest_div).
__device__ __forceinline__ double dvr(double a, double d, double r) {
    const double q0 = __dmul_rn(a, r);
    const double q1 = __fma_rn(__fma_rn(-q0, d, a), r, q0);
    const double q2 = __fma_rn(__fma_rn(-q1, d, a), r, q1);
    return a == 0.0 ? q0 : q2;
}

// Boundary rule codes (PKG/boundary.py:22-34)
enum BcKind : int { BC_DIRICHLET = 0, BC_NEUMANN = 1, BC_PERIODIC = 2 };

struct BcSpec {
    int kind[3][2];
    double val[3][2];
};

// ---------------------------------------------------------------------------
// Natural (reference) layout: C-order array with element strides.  `core`
// points at core index (0,0,0): array index == grid index
// (PKG/grid.py:199-208).
// ---------------------------------------------------------------------------
struct NatView {
    double* core;
    long st[3];
};

// ---------------------------------------------------------------------------
// Ghost semantics of fill_ghosts (PKG/boundary.py:90-156) evaluated
// point-wise.  Passes run from the last axis to the first, so the value held
// at a point outside the interior is produced by the pass of the LOWEST axis
// that writes it, applied to the (already final) mirror value.  We walk that
// chain and evaluate the recorded rules innermost-first, reproducing the
// reference's exact sequence of `2.0 * v - mirror` operations.
//
// Index convention: core indices, halo g >= 1 handled by callers for the
// natural fill (ring r); the solver uses halo 1 only.
// ---------------------------------------------------------------------------
struct AxisGeo {
    int m;       // cells along the axis (grid shape)
    int edge;    // 1 if the field is edge-centered along this axis
    int iface = 0;  // slab interfaces (bit 0 lo, bit 1 hi): the rows beyond
                    // hold a neighbour's data, not ghosts (fill_ghosts_slab)
};

// Is core index x along an axis "owned" (written) by that axis' pass?
// cell axis: ghosts 0 and m+1 (and further rings).  edge axis: the high wall
// m (always) and the low wall 0 unless periodic (never written, PKG/
// boundary.py:117-125), plus rings beyond the walls.
__device__ __forceinline__ bool owned(const AxisGeo& a, int lo_kind, int x) {
    if ((a.iface & 1) && x <= 0) return false;
    if ((a.iface & 2) && x >= (a.edge ? a.m : a.m + 1)) return false;
    if (!a.edge) return x <= 0 || x >= a.m + 1;
    if (x >= a.m) return true;
    if (x < 0) return true;
    if (x == 0) return lo_kind != BC_PERIODIC;
    return false;
}

// One step of the chain: given an owned index x along an axis, rewrite x to
// its mirror and report the operation: 0 = copy, 1 = 2v - mirror,
// 2 = constant v (terminates).
__device__ __forceinline__ int rule_step(const AxisGeo& a, const BcSpec& bc,
                                         int axis, int& x, double& v) {
    const int m = a.m;
    if (!a.edge) {
        // core index x <= 0: lo ring r = 1 - x (core 0 == data g-1 == ring 1)
        if (x <= 0) {
            int r = 1 - x;
            int k = bc.kind[axis][0];
            v = bc.val[axis][0];
            if (k == BC_DIRICHLET) { x = r; return 1; }      // lo_mirror g+r-1
            if (k == BC_NEUMANN) { x = r; return 0; }
            x = m + 1 - r;                                   // g+m-r
            return 0;
        } else {
            int r = x - m;                                   // x = m + r
            int k = bc.kind[axis][1];
            v = bc.val[axis][1];
            if (k == BC_DIRICHLET) { x = m + 1 - r; return 1; }  // hi_mirror
            if (k == BC_NEUMANN) { x = m + 1 - r; return 0; }
            x = r;                                           // g+r-1
            return 0;
        }
    }
    // edge axis: walls at 0 and m, rings beyond
    if (x == m) {
        int k = bc.kind[axis][1];
        v = bc.val[axis][1];
        if (k == BC_DIRICHLET) return 2;
        if (k == BC_NEUMANN) { x = m - 1; return 0; }
        x = 0;                                               // hi wall = lo wall
        return 0;
    }
    if (x == 0) {  // lo wall, non-periodic
        int k = bc.kind[axis][0];
        v = bc.val[axis][0];
        if (k == BC_DIRICHLET) return 2;
        x = 1;                                               // neumann copy
        return 0;
    }
    if (x < 0) {
        int r = -x;
        int k = bc.kind[axis][0];
        v = bc.val[axis][0];
        if (k == BC_DIRICHLET) { x = r; return 1; }          // 2v - data[b_lo+r]
        if (k == BC_NEUMANN) { x = r; return 0; }
        x = m - r;                                           // data[b_hi - r]
        return 0;
    }
    // x > m
    int r = x - m;
    int k = bc.kind[axis][1];
    v = bc.val[axis][1];
    if (k == BC_DIRICHLET) { x = m - r; return 1; }
    if (k == BC_NEUMANN) { x = m - r; return 0; }
    x = r;                                                   // data[b_lo + r]
    return 0;
}

// Resolve the value at core index x[0..dim) given a reader of raw stored
// values (interior points, or the never-written periodic low wall).
template <int DIM, class Reader>
__device__ __forceinline__ double ghost_value(const AxisGeo* ax, const BcSpec& bc,
                                              int x0, int x1, int x2,
                                              const Reader& rd) {
    int x[3] = {x0, x1, x2};
    int op[3];
    double vv[3];
    int nop = 0;
    double term_v = 0.0;
    bool terminal = false;
#pragma unroll 1
    for (int guard = 0; guard < 3; ++guard) {
        int a = -1;
#pragma unroll
        for (int t = 0; t < DIM; ++t) {
            if (owned(ax[t], bc.kind[t][0], x[t])) { a = t; break; }
        }
        if (a < 0) break;
        double v;
        int o = rule_step(ax[a], bc, a, x[a], v);
        if (o == 2) { terminal = true; term_v = v; break; }
        op[nop] = o;
        vv[nop] = v;
        ++nop;
    }
    double val = terminal ? term_v : rd(x[0], x[1], x[2]);
    for (int t = nop - 1; t >= 0; --t)
        if (op[t] == 1) val = sb(ml(2.0, vv[t]), val);
    return val;
}

}  // namespace fasmg
