// fasmg_stencil.cuh -- branch-free stencil kernels on the parity-blocked
// layout (included by fasmg_engine.cu, which defines Lvl/at/qbit).
//
// Ghost pads.  Every class array carries pad blocks 0 and B+1 per axis.  A
// 5/7-point stencil reads a ghost only as the neighbor of the one interior
// point it mirrors, so the pad slot of each boundary point's ghost (and the
// edge-axis wall slots) are kept current: the kernel that writes a
// boundary point also writes the ghost value the reference's fill_ghosts
// would produce from it (PKG/boundary.py:110-156):
//   cell axis   lo ghost (x=0)   : dirichlet 2v - p(1), neumann p(1),
//                                  periodic p(n)
//               hi ghost (x=n+1) : dirichlet 2v - p(n), neumann p(n),
//                                  periodic p(1)
//   edge axis   lo wall (x=0)    : dirichlet v, neumann p(1), periodic the
//                                  stored wall (never written)
//               hi wall (x=n)    : dirichlet v, neumann p(n-1), periodic =
//                                  lo wall
// In the blocked layout these are exactly the slots a branch-free neighbor
// load hits: W of (q=1, b=1) is (q=0, b=0); E of (q=0, b=B) is (q=1, b=B+1);
// E of the edge point (q=1, b=B) is the wall slot (q=0, b=B).  A pad slot is
// only ever read by the point it mirrors, so a kernel may write it in the
// same launch after that thread's own loads.
#pragma once

// (included inside namespace fasmg)

// linear strides of the block axes
template <int D>
__device__ __forceinline__ long bstride(const Lvl& L, int a) {
    if (D == 3) return a == 0 ? L.s0 : (a == 1 ? L.s1 : 1);
    return a == 0 ? L.s0 : 1;
}

// 3D-block thread mapping: x -> last block axis, y -> next, z -> axis 0.
template <int D>
__device__ __forceinline__ bool tile_coords(const Lvl& L, int* bb) {
    if (D == 3) {
        bb[2] = blockIdx.x * blockDim.x + threadIdx.x + 1;
        bb[1] = blockIdx.y * blockDim.y + threadIdx.y + 1;
        bb[0] = blockIdx.z * blockDim.z + threadIdx.z + 1;
        return bb[0] <= L.B[0] && bb[1] <= L.B[1] && bb[2] <= L.B[2];
    }
    bb[1] = blockIdx.x * blockDim.x + threadIdx.x + 1;
    bb[0] = blockIdx.y * blockDim.y + threadIdx.y + 1;
    bb[2] = 0;
    return bb[0] <= L.B[0] && bb[1] <= L.B[1];
}

// global block index along axis 0 (slab decomposition: local + offset)
__device__ __forceinline__ int gb0(const Lvl& L, const int* bb) { return bb[0] + L.off0; }

// is the block on the GLOBAL boundary of the level?  (axis 0 uses the
// global index, so internal slab faces are not boundaries)
template <int D>
__device__ __forceinline__ bool on_boundary(const Lvl& L, const int* bb) {
    const int g = gb0(L, bb);
    bool r = g == 1 || g == L.G0;
#pragma unroll
    for (int a = 1; a < D; ++a) r = r || bb[a] == 1 || bb[a] == L.B[a];
    return r;
}

// edge-axis wall position of class c at block bb (not an unknown)
template <int D, int EA>
__device__ __forceinline__ bool is_wall(const Lvl& L, int c, const int* bb) {
    if (EA < 0) return false;
    const int g = EA == 0 ? gb0(L, bb) : bb[EA];
    const int B = EA == 0 ? L.G0 : L.B[EA];
    return qbit<D>(c, EA) == 0 && g == B;
}

// sum of the 2d neighbors of point (c, o) in the reference order
// ((((E+W)+N)+S)+T)+B, all through (pad-backed) branch-free loads.
template <int D>
__device__ __forceinline__ double nsum_fast(const double* __restrict__ P, const Lvl& L, int c,
                                            long o) {
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        const int bit = 1 << (D - 1 - a);
        const long dcls = (long)((c ^ bit) - c) * L.cls;
        const long sa = bstride<D>(L, a);
        const bool q = (c & bit) != 0;
        const double e = P[o + dcls + (q ? 0 : sa)];
        const double w = P[o + dcls - (q ? sa : 0)];
        s = (a == 0) ? ad(e, w) : ad(ad(s, e), w);
    }
    return s;
}

// After writing value v at boundary point (c, bb) (offset o), refresh the
// ghost / wall slots derived from it.
template <int D, int EA>
__device__ __forceinline__ void write_pads(double* __restrict__ P, const Lvl& L,
                                           const BcSpec& bc, int c, const int* bb, long o,
                                           double v) {
#pragma unroll
    for (int a = 0; a < D; ++a) {
        const int bit = 1 << (D - 1 - a);
        const long dcls = (long)((c ^ bit) - c) * L.cls;
        const long sa = bstride<D>(L, a);
        const bool q = (c & bit) != 0;
        const int B = a == 0 ? L.G0 : L.B[a];   // global extent (axis 0 may be a slab)
        const int g = a == 0 ? gb0(L, bb) : bb[a];
        if (a != EA) {
            if (q && g == 1) {
                const int k = bc.kind[a][0];
                if (k == BC_DIRICHLET) P[o + dcls - sa] = sb(ml(2.0, bc.val[a][0]), v);
                else if (k == BC_NEUMANN) P[o + dcls - sa] = v;
                else P[o + (long)B * sa] = v;  // periodic: hi ghost x=n+1 <- p(1)
            }
            if (!q && g == B) {
                const int k = bc.kind[a][1];
                if (k == BC_DIRICHLET) P[o + dcls + sa] = sb(ml(2.0, bc.val[a][1]), v);
                else if (k == BC_NEUMANN) P[o + dcls + sa] = v;
                else P[o - (long)B * sa] = v;  // periodic: lo ghost x=0 <- p(n)
            }
        } else {
            if (q && g == 1 && bc.kind[a][0] == BC_NEUMANN) P[o + dcls - sa] = v;
            if (q && g == B && bc.kind[a][1] == BC_NEUMANN) P[o + dcls] = v;
        }
    }
}

// ------------------------------------------------------ fused halo push
// Slab ranks (multi-GPU): the neighbours' halo planes of this level's array
// (peer memory over NVLink, or the same device for virtual ranks).  A sweep
// that writes a point of its first/last local block plane also stores it
// straight into the neighbour's halo plane -- the exchange of the updated
// classes is fused into the compute kernel (no separate push launch); the
// host then only publishes the release/acquire counter.  q0=0 classes of
// plane B0 feed the upper rank's plane 0, q0=1 classes of plane 1 the lower
// rank's plane B0+1 (the same routing as k_push_plane).
struct PeerHalo {
    double* lo = nullptr;
    double* hi = nullptr;
};

template <int D>
__device__ __forceinline__ void push_halo(const PeerHalo& ph, const Lvl& L, int c, const int* bb,
                                          double v) {
    constexpr int BIT0 = 1 << (D - 1);
    if (ph.hi && !(c & BIT0) && bb[0] == L.B[0]) {
        ph.hi[at<D>(L, c, 0, bb[1], bb[2])] = v;
        __threadfence_system();
    }
    if (ph.lo && (c & BIT0) && bb[0] == 1) {
        ph.lo[at<D>(L, c, L.B[0] + 1, bb[1], bb[2])] = v;
        __threadfence_system();
    }
}

// ------------------------------------------------------------- pad fill
// Initialize every pad/wall slot of a level from its interior (after a
// pack, a restriction or an edge correction).  Launch: grid.y = face id
// (2*D faces), x over the face's blocks.
template <int D, int EA>
__device__ __forceinline__ void pad_fill_pt(double* __restrict__ P, const Lvl& L,
                                            const BcSpec& bc, int face, int i1, int i2) {
    const int a = face >> 1, side = face & 1;
    // the other axes' blocks: (i1, i2) 0-based along oth[0], oth[1]
    int oth[2], no = 0;
#pragma unroll
    for (int t = 0; t < D; ++t)
        if (t != a) oth[no++] = t;
    if (i1 >= L.B[oth[0]] || (D == 3 ? i2 >= L.B[oth[1]] : i2 > 0)) return;
    if (a == 0 && ((side == 0 && L.off0 != 0) || (side == 1 && L.off0 + L.B[0] != L.G0)))
        return;  // internal slab face: the halo comes from the neighbor rank
    int bb[3] = {0, 0, 0};
    bb[a] = side ? L.B[a] : 1;
    bb[oth[0]] = 1 + i1;
    if (D == 3) bb[oth[1]] = 1 + i2;
    const long o0 = at<D>(L, 0, bb[0], bb[1], bb[2]);
    // every class's value first: the loads go out together instead of one
    // L2 round trip per class behind the previous class's pad stores (no
    // slot read here is written below: a wall slot written for class c is
    // skipped as c's own point)
    double pv[1 << D];
#pragma unroll
    for (int c = 0; c < (1 << D); ++c) pv[c] = P[o0 + (long)c * L.cls];
#pragma unroll
    for (int c = 0; c < (1 << D); ++c) {
        const long o = o0 + (long)c * L.cls;
        if (EA >= 0 && a == EA && qbit<D>(c, EA) == 0) {
            const long sa = bstride<D>(L, EA);
            // constant walls of this class at this face
            if (side == 0) {
                if (bc.kind[EA][0] == BC_DIRICHLET) P[o - sa] = bc.val[EA][0];
            } else {
                // o is the hi wall slot itself (q=0, b=B)
                if (bc.kind[EA][1] == BC_DIRICHLET) P[o] = bc.val[EA][1];
                else if (bc.kind[EA][1] == BC_PERIODIC) P[o] = P[o - (long)L.B[EA] * sa];
            }
        }
        if (is_wall<D, EA>(L, c, bb)) continue;
        write_pads<D, EA>(P, L, bc, c, bb, o, pv[c]);
    }
}

// grid: x over the face's last other axis (3D; 2D: the other axis), y over
// the first other axis (3D), z = face -- no integer division
template <int D, int EA>
__global__ void k_pad_fill(double* __restrict__ P, Lvl L, BcSpec bc) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (D == 3) pad_fill_pt<D, EA>(P, L, bc, blockIdx.z, blockIdx.y, i);
    else pad_fill_pt<D, EA>(P, L, bc, blockIdx.z, i, 0);
}

// ------------------------------------------------------------- smoothing
// One launch = the reference's colors whose classes are in MASK (mutually
// independent classes; PKG/smoothers.py:136-153).  Thread per block.
template <int D, int EA, unsigned MASK>
__device__ __forceinline__ void sweep_pt(double* __restrict__ P, const double* __restrict__ F,
                                         const Lvl& L, const BcSpec& bc, const int* bb,
                                         const PeerHalo& ph = PeerHalo()) {
    const long o0 = at<D>(L, 0, bb[0], bb[1], bb[2]);
    constexpr int NC = 1 << D;
    // phase 1: issue every load of every class before any arithmetic, so
    // the division's slow-path call cannot serialize them
    double nbv[NC][2 * D], fv[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        if (!((MASK >> c) & 1u)) continue;
        const long o = o0 + (long)c * L.cls;
        fv[c] = F[o];
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const int bit = 1 << (D - 1 - a);
            const long dcls = (long)((c ^ bit) - c) * L.cls;
            const long sa = bstride<D>(L, a);
            const bool q = (c & bit) != 0;
            // opposite-parity classes are not written by this launch except
            // pad slots only this thread reads (before writing): the
            // non-coherent read-only path is safe
            nbv[c][2 * a] = __ldg(P + o + dcls + (q ? 0 : sa));
            nbv[c][2 * a + 1] = __ldg(P + o + dcls - (q ? sa : 0));
        }
    }
    // phase 2: numerators h2*f + b*((((E+W)+N)+S)+T)+B for every class first
    // (so the loaded values are dead before any division's slow-path call),
    // then the IEEE divisions by denom (KER/numpy_backend.py:44,62)
    double nv[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        if (!((MASK >> c) & 1u)) continue;
        double ns = ad(nbv[c][0], nbv[c][1]);
#pragma unroll
        for (int t = 2; t < 2 * D; ++t) ns = ad(ns, nbv[c][t]);
        nv[c] = ad(ml(L.h2, fv[c]), ml(L.b, ns));
    }
#pragma unroll
    for (int c = 0; c < NC; ++c)
        if ((MASK >> c) & 1u) nv[c] = dvr(nv[c], L.denom, L.rden);
    const bool bnd = on_boundary<D>(L, bb);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        if (!((MASK >> c) & 1u)) continue;
        if (is_wall<D, EA>(L, c, bb)) continue;
        const long o = o0 + (long)c * L.cls;
        P[o] = nv[c];
        if (bnd) write_pads<D, EA>(P, L, bc, c, bb, o, nv[c]);
        push_halo<D>(ph, L, c, bb, nv[c]);
    }
}

template <int D, int EA, unsigned MASK, int MINB = 3>
__global__ void __launch_bounds__(256, MINB) k_sweep_fast(double* __restrict__ P,
                                                    const double* __restrict__ F, Lvl L,
                                                    BcSpec bc, PeerHalo ph = PeerHalo()) {
    int bb[3];
    if (!tile_coords<D>(L, bb)) return;
    sweep_pt<D, EA, MASK>(P, F, L, bc, bb, ph);
}

// Same update, one thread per (block, class): grid.z enumerates (b0, k-th
// class of MASK) [3D] / (k-th class) [2D].  Fewer registers per thread and
// one division each, so many more warps are resident to hide DRAM latency;
// the classes of one block share their loads through L1/L2.
template <int D, unsigned MASK>
__device__ __forceinline__ int mask_class(int k) {
    int n = 0;
#pragma unroll
    for (int c = 0; c < (1 << D); ++c)
        if ((MASK >> c) & 1u) {
            if (n == k) return c;
            ++n;
        }
    return 0;
}

template <int D, int EA, unsigned MASK>
__global__ void __launch_bounds__(256) k_sweep_pc(double* __restrict__ P,
                                                  const double* __restrict__ F, Lvl L,
                                                  BcSpec bc) {
    constexpr int NCM = __builtin_popcount(MASK);
    int bb[3], kc;
    if (D == 3) {
        bb[2] = blockIdx.x * blockDim.x + threadIdx.x + 1;
        bb[1] = blockIdx.y * blockDim.y + threadIdx.y + 1;
        bb[0] = blockIdx.z / NCM + 1;
        kc = blockIdx.z % NCM;
        if (bb[1] > L.B[1] || bb[2] > L.B[2]) return;
    } else {
        bb[1] = blockIdx.x * blockDim.x + threadIdx.x + 1;
        bb[0] = blockIdx.y * blockDim.y + threadIdx.y + 1;
        bb[2] = 0;
        kc = blockIdx.z;
        if (bb[0] > L.B[0] || bb[1] > L.B[1]) return;
    }
    const int c = mask_class<D, MASK>(kc);
    if (is_wall<D, EA>(L, c, bb)) return;
    const long o = at<D>(L, c, bb[0], bb[1], bb[2]);
    double nbv[2 * D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        const int bit = 1 << (D - 1 - a);
        const long dcls = (long)((c ^ bit) - c) * L.cls;
        const long sa = bstride<D>(L, a);
        const bool q = (c & bit) != 0;
        nbv[2 * a] = P[o + dcls + (q ? 0 : sa)];
        nbv[2 * a + 1] = P[o + dcls - (q ? sa : 0)];
    }
    const double fv = F[o];
    double ns = ad(nbv[0], nbv[1]);
#pragma unroll
    for (int t = 2; t < 2 * D; ++t) ns = ad(ns, nbv[t]);
    const double v = dvr(ad(ml(L.h2, fv), ml(L.b, ns)), L.denom, L.rden);
    P[o] = v;
    if (on_boundary<D>(L, bb)) write_pads<D, EA>(P, L, bc, c, bb, o, v);
}

// 2.5D marching half-sweep.  Each thread owns one column of blocks along
// axis 0 (a chunk of planes) and keeps, for every opposite-parity class k, a
// two-plane register window of its values along axis 0: classes with
// q0(k)=0 hold planes (b0-1, b0), classes with q0(k)=1 hold (b0, b0+1) --
// exactly the W/E neighbors along axis 0 of the updated classes.  The next
// plane of the window and of f is prefetched one step ahead, so every warp
// keeps independent DRAM loads in flight across the whole column.  Axis-1/2
// neighbors come from L1 (loaded as window values by neighboring threads).
template <int D>
__host__ __device__ constexpr unsigned opp_mask(unsigned m) {
    unsigned r = 0;
    for (int c = 0; c < (1 << D); ++c)
        if ((m >> c) & 1u)
            for (int a = 0; a < D; ++a) r |= 1u << (c ^ (1 << (D - 1 - a)));
    return r;
}

template <int D, int EA, unsigned MASK>
__global__ void __launch_bounds__(256) k_sweep_march(double* __restrict__ P,
                                                     const double* __restrict__ F, Lvl L,
                                                     BcSpec bc, int chunk) {
    constexpr int NC = 1 << D;
    constexpr unsigned OPP = opp_mask<D>(MASK);
    constexpr int BIT0 = 1 << (D - 1);
    int bb[3];
    int z;
    if (D == 3) {
        bb[2] = blockIdx.x * blockDim.x + threadIdx.x + 1;
        bb[1] = blockIdx.y * blockDim.y + threadIdx.y + 1;
        z = blockIdx.z;
        if (bb[1] > L.B[1] || bb[2] > L.B[2]) return;
    } else {
        bb[1] = blockIdx.x * blockDim.x + threadIdx.x + 1;
        bb[2] = 0;
        z = blockIdx.y;
        if (bb[1] > L.B[1]) return;
    }
    const int b0s = 1 + z * chunk;
    const int b0e = min(L.B[0], b0s + chunk - 1);
    const long s0 = L.s0;
    const long col = at<D>(L, 0, 0, bb[1], bb[2]);  // class 0, plane 0
    bool bnd_col = false;
#pragma unroll
    for (int a = 1; a < D; ++a) bnd_col = bnd_col || bb[a] == 1 || bb[a] == L.B[a];

    double w0[NC], w1[NC], wn[NC], fv[NC], fn[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        if (!((OPP >> k) & 1u)) continue;
        const long ok = col + (long)k * L.cls;
        const int lo = (k & BIT0) ? b0s : b0s - 1;
        w0[k] = P[ok + (long)lo * s0];
        w1[k] = P[ok + (long)(lo + 1) * s0];
    }
#pragma unroll
    for (int c = 0; c < NC; ++c)
        if ((MASK >> c) & 1u) fv[c] = F[col + (long)c * L.cls + (long)b0s * s0];

    for (int b0 = b0s; b0 <= b0e; ++b0) {
        const bool more = b0 < b0e;
        if (more) {  // prefetch the next step's window plane and f
#pragma unroll
            for (int k = 0; k < NC; ++k) {
                if (!((OPP >> k) & 1u)) continue;
                const int nxt = (k & BIT0) ? b0 + 2 : b0 + 1;
                wn[k] = P[col + (long)k * L.cls + (long)nxt * s0];
            }
#pragma unroll
            for (int c = 0; c < NC; ++c)
                if ((MASK >> c) & 1u) fn[c] = F[col + (long)c * L.cls + (long)(b0 + 1) * s0];
        }
        bb[0] = b0;
        const long pl = col + (long)b0 * s0;
        double nv[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            if (!((MASK >> c) & 1u)) continue;
            const int k0 = c ^ BIT0;
            // ((((E+W)+N)+S)+T)+B  (KER/numpy_backend.py:44,62)
            double ns = ad(w1[k0], w0[k0]);
#pragma unroll
            for (int a = 1; a < D; ++a) {
                const int bit = 1 << (D - 1 - a);
                const long sa = bstride<D>(L, a);
                const bool q = (c & bit) != 0;
                const long ok = pl + (long)(c ^ bit) * L.cls;
                const double e = P[ok + (q ? 0 : sa)];
                const double w = P[ok - (q ? sa : 0)];
                ns = ad(ad(ns, e), w);
            }
            nv[c] = dvr(ad(ml(L.h2, fv[c]), ml(L.b, ns)), L.denom, L.rden);
        }
        const bool bnd = bnd_col || b0 + L.off0 == 1 || b0 + L.off0 == L.G0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            if (!((MASK >> c) & 1u)) continue;
            if (is_wall<D, EA>(L, c, bb)) continue;
            const long o = pl + (long)c * L.cls;
            P[o] = nv[c];
            if (bnd) write_pads<D, EA>(P, L, bc, c, bb, o, nv[c]);
        }
        if (more) {
#pragma unroll
            for (int k = 0; k < NC; ++k) {
                if (!((OPP >> k) & 1u)) continue;
                w0[k] = w1[k];
                w1[k] = wn[k];
            }
#pragma unroll
            for (int c = 0; c < NC; ++c)
                if ((MASK >> c) & 1u) fv[c] = fn[c];
        }
    }
}

// 2.5D marching half-sweep staged through shared memory (3D, large levels).
// A CTA owns a 32 (b2) x 8 (b1) tile of block columns and marches a chunk
// of planes along b0.  For each opposite-parity class it keeps a ring of 3
// plane tiles (with a 1-block in-plane halo) in shared memory: two planes
// are the class's current axis-0 window, the third is being filled by
// cp.async for the next step, so DRAM loads stay in flight independently of
// registers.  f is prefetched one plane ahead in registers.  Arithmetic and
// pad maintenance are those of k_sweep_fast.
namespace smem_sweep {
constexpr int TX = 32, TY = 8, RX = TX + 2, RY = TY + 2, PL = RX * RY, RING = 3;
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int EA, unsigned MASK>
__global__ void __launch_bounds__(256) k_sweep_smem(double* __restrict__ P,
                                                    const double* __restrict__ F, Lvl L,
                                                    BcSpec bc, int chunk) {
    using namespace smem_sweep;
    constexpr int D = 3, NC = 8;
    constexpr unsigned OPP = opp_mask<3>(MASK);
    extern __shared__ double sm[];  // [4 opp classes][RING][PL]
    // opposite class -> ring index (compile time)
    auto ridx = [](int k) {
        int n = 0;
        for (int t = 0; t < k; ++t) n += (OPP >> t) & 1u;
        return n;
    };
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
    const int x0 = blockIdx.x * TX + 1, y0 = blockIdx.y * TY + 1;
    const int b0s = 1 + blockIdx.z * chunk;
    const int b0e = min(L.B[0], b0s + chunk - 1);
    int bb[3];
    bb[2] = x0 + tx;
    bb[1] = y0 + ty;
    const bool active = bb[1] <= L.B[1] && bb[2] <= L.B[2];
    const long s0 = L.s0, s1 = L.s1;

    auto load_plane = [&](int k, int pb) {
        double* dst = sm + (ridx(k) * RING + (pb % RING)) * PL;
        const double* src = P + (long)k * L.cls + (long)pb * s0 + OFF;
        for (int e = tid; e < PL; e += TX * TY) {
            const int r = e / RX, cx = e - r * RX;
            const int gb1 = min(y0 - 1 + r, L.B[1] + 1);
            const int gb2 = min(x0 - 1 + cx, L.B[2] + 1);
            cp_async8(dst + e, src + (long)gb1 * s1 + gb2);
        }
    };
    // prologue: both window planes of every opposite class
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        if (!((OPP >> k) & 1u)) continue;
        const int lo = (k & 4) ? b0s : b0s - 1;
        load_plane(k, lo);
        load_plane(k, lo + 1);
    }
    cp_async_commit();
    const long col = active ? at<D>(L, 0, 0, bb[1], bb[2]) : 0;
    double fv[NC], fn[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c)
        if ((MASK >> c) & 1u) fv[c] = active ? __ldg(F + col + (long)c * L.cls + (long)b0s * s0) : 0.0;

    for (int b0 = b0s; b0 <= b0e; ++b0) {
        const bool more = b0 < b0e;
        if (more) {
#pragma unroll
            for (int k = 0; k < NC; ++k) {
                if (!((OPP >> k) & 1u)) continue;
                const int lo = (k & 4) ? b0 : b0 - 1;
                load_plane(k, lo + 2);
            }
            cp_async_commit();
#pragma unroll
            for (int c = 0; c < NC; ++c)
                if ((MASK >> c) & 1u)
                    fn[c] = active ? __ldg(F + col + (long)c * L.cls + (long)(b0 + 1) * s0) : 0.0;
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        if (active) {
            bb[0] = b0;
            const long pl = col + (long)b0 * s0;
            const int ci = (ty + 1) * RX + (tx + 1);
            double nv[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                if (!((MASK >> c) & 1u)) continue;
                // axis 0: window (lo, lo+1) of class c^4 -> E = lo+1, W = lo
                const int k0 = c ^ 4;
                const int lo0 = (k0 & 4) ? b0 : b0 - 1;
                const double* w0 = sm + ridx(k0) * RING * PL;
                double ns = ad(w0[((lo0 + 1) % RING) * PL + ci], w0[(lo0 % RING) * PL + ci]);
                // axis 1 (b1 = rows), class c^2 at plane b0
                {
                    const int k1 = c ^ 2;
                    const double* w = sm + (ridx(k1) * RING + (b0 % RING)) * PL;
                    const bool q = (c & 2) != 0;
                    const double e = w[ci + (q ? 0 : RX)];
                    const double wv = w[ci - (q ? RX : 0)];
                    ns = ad(ad(ns, e), wv);
                }
                // axis 2 (b2 = cols), class c^1 at plane b0
                {
                    const int k2 = c ^ 1;
                    const double* w = sm + (ridx(k2) * RING + (b0 % RING)) * PL;
                    const bool q = (c & 1) != 0;
                    const double e = w[ci + (q ? 0 : 1)];
                    const double wv = w[ci - (q ? 1 : 0)];
                    ns = ad(ad(ns, e), wv);
                }
                nv[c] = ad(ml(L.h2, fv[c]), ml(L.b, ns));
            }
#pragma unroll
            for (int c = 0; c < NC; ++c)
                if ((MASK >> c) & 1u) nv[c] = dvr(nv[c], L.denom, L.rden);
            const bool bnd = on_boundary<3>(L, bb);
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                if (!((MASK >> c) & 1u)) continue;
                if (is_wall<D, EA>(L, c, bb)) continue;
                const long o = pl + (long)c * L.cls;
                P[o] = nv[c];
                if (bnd) write_pads<D, EA>(P, L, bc, c, bb, o, nv[c]);
            }
        }
        __syncthreads();  // the next prefetch overwrites the oldest ring slot
        if (more) {
#pragma unroll
            for (int c = 0; c < NC; ++c)
                if ((MASK >> c) & 1u) fv[c] = fn[c];
        }
    }
}

// a*c - b*((nsum - 2d c) * inv_h2) at (c, o)  (KER/numpy_backend.py:69-99)
template <int D>
__device__ __forceinline__ double op_fast(const double* __restrict__ P, const Lvl& L, int c,
                                          long o) {
    const double cv = P[o];
    const double ns = nsum_fast<D>(P, L, c, o);
    const double lap = ml(sb(ns, ml(D == 3 ? 6.0 : 4.0, cv)), L.inv_h2);
    return sb(ml(L.a, cv), ml(L.b, lap));
}

// coarse cell of fine block bb: the fine block's GLOBAL index I is the
// coarse cell index; coarse class bit I&1, coarse block (I+1)>>1, made
// local to the coarse level's slab (Lc.off0)
template <int D>
__device__ __forceinline__ void coarse_of(const Lvl& L, const Lvl& Lc, const int* bb, int& cc,
                                          int* cb) {
    cc = 0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        const int I = a == 0 ? gb0(L, bb) : bb[a];
        cc |= (I & 1) << (D - 1 - a);
        cb[a] = ((I + 1) >> 1) - (a == 0 ? Lc.off0 : 0);
    }
}

// ----------------------------------------------------------- tau kernel
// Cell-centered fine level k -> coarse level k+1 in one pass: residual at the
// 2^d children of coarse cell bb, restriction of r and p (lexicographic child
// order = descending class id, KER/numba_backend.py:222-253), stored into the
// coarse level's blocked arrays with its ghost pads (full BC on p_c,
// PKG/fas.py:99-107).
template <int D>
__device__ __forceinline__ void tau_pt(const double* __restrict__ P, const double* __restrict__ F,
                                       const Lvl& L, double* __restrict__ Pc,
                                       double* __restrict__ Fc, const Lvl& Lc, const BcSpec& bc,
                                       const int* bb, double* __restrict__ PIc = nullptr) {
    constexpr int NC = 1 << D;
    const long o0 = at<D>(L, 0, bb[0], bb[1], bb[2]);
    // phase 1: all loads (2^d centers, 2^d f, and the d*2^(d-1) neighbors
    // outside the block) before any arithmetic
    double pc[NC], fv[NC], out[NC][D];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const long o = o0 + (long)c * L.cls;
        pc[c] = __ldg(P + o);
        fv[c] = __ldg(F + o);
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const int bit = 1 << (D - 1 - a);
            const long dcls = (long)((c ^ bit) - c) * L.cls;
            const long sa = bstride<D>(L, a);
            // the neighbor across the block face: W of q=1, E of q=0
            out[c][a] = (c & bit) ? __ldg(P + o + dcls - sa) : __ldg(P + o + dcls + sa);
        }
    }
    // phase 2: residual at every child in the reference order, restriction
    // in lexicographic child order (descending class id)
    double rp = 0.0, rr = 0.0;
#pragma unroll
    for (int c = NC - 1; c >= 0; --c) {
        double ns = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const int bit = 1 << (D - 1 - a);
            const double inside = pc[c ^ bit];
            const double e = (c & bit) ? inside : out[c][a];
            const double w = (c & bit) ? out[c][a] : inside;
            ns = a == 0 ? ad(e, w) : ad(ad(ns, e), w);
        }
        const double lap = ml(sb(ns, ml(D == 3 ? 6.0 : 4.0, pc[c])), L.inv_h2);
        const double r = sb(fv[c], sb(ml(L.a, pc[c]), ml(L.b, lap)));
        if (c == NC - 1) { rp = pc[c]; rr = r; }
        else { rp = ad(rp, pc[c]); rr = ad(rr, r); }
    }
    const double sc = D == 3 ? 0.125 : 0.25;
    int cc = 0, cb[3] = {0, 0, 0};
    coarse_of<D>(L, Lc, bb, cc, cb);
    const long oc = at<D>(Lc, cc, cb[0], cb[1], cb[2]);
    const double pcv = ml(rp, sc);
    Pc[oc] = pcv;
    if (PIc) PIc[oc] = pcv;  // pinit, for the fused correction
    Fc[oc] = ml(rr, sc);
    if (on_boundary<D>(Lc, cb)) write_pads<D, -1>(Pc, Lc, bc, cc, cb, oc, pcv);
}

template <int D>
__global__ void __launch_bounds__(256) k_tau_fast(const double* __restrict__ P,
                                                  const double* __restrict__ F, Lvl L,
                                                  double* __restrict__ Pc,
                                                  double* __restrict__ Fc, Lvl Lc, BcSpec bc,
                                                  double* __restrict__ PIc = nullptr) {
    int bb[3];
    if (!tile_coords<D>(L, bb)) return;
    tau_pt<D>(P, F, L, Pc, Fc, Lc, bc, bb, PIc);
}

// f_c += a*p_c - b*Lap(p_c) on the coarse level (PKG/fas.py:108-110)
template <int D, int EA>
__device__ __forceinline__ void coarse_src_pt(const double* __restrict__ Pc,
                                              double* __restrict__ Fc, const Lvl& L,
                                              const int* bb) {
    const long o0 = at<D>(L, 0, bb[0], bb[1], bb[2]);
#pragma unroll
    for (int c = 0; c < (1 << D); ++c) {
        if (is_wall<D, EA>(L, c, bb)) continue;
        const long o = o0 + (long)c * L.cls;
        Fc[o] = ad(Fc[o], op_fast<D>(Pc, L, c, o));
    }
}

template <int D, int EA>
__global__ void __launch_bounds__(256) k_coarse_src_fast(const double* __restrict__ Pc,
                                                         double* __restrict__ Fc, Lvl L) {
    int bb[3];
    if (!tile_coords<D>(L, bb)) return;
    coarse_src_pt<D, EA>(Pc, Fc, L, bb);
}

// Cell-centered coarse correction (PKG/fas.py:119-123): c = p_c - R(p), R(p)
// recomputed from the unchanged fine p (equals the reference's pinit),
// injected and added; refreshes the fine ghost pads.
template <int D>
__device__ __forceinline__ void correct_pt(double* __restrict__ P, const Lvl& L,
                                           const double* __restrict__ Pc, const Lvl& Lc,
                                           const BcSpec& bc, const int* bb) {
    const long o0 = at<D>(L, 0, bb[0], bb[1], bb[2]);
    double pv[1 << D];
    double rp = 0.0;
#pragma unroll
    for (int c = (1 << D) - 1; c >= 0; --c) {
        pv[c] = P[o0 + (long)c * L.cls];
        rp = (c == (1 << D) - 1) ? pv[c] : ad(rp, pv[c]);
    }
    rp = ml(rp, D == 3 ? 0.125 : 0.25);
    int cc = 0, cb[3] = {0, 0, 0};
    coarse_of<D>(L, Lc, bb, cc, cb);
    const double corr = sb(Pc[at<D>(Lc, cc, cb[0], cb[1], cb[2])], rp);
    const bool bnd = on_boundary<D>(L, bb);
#pragma unroll
    for (int c = 0; c < (1 << D); ++c) {
        const long o = o0 + (long)c * L.cls;
        const double v = ad(pv[c], corr);
        P[o] = v;
        if (bnd) write_pads<D, -1>(P, L, bc, c, bb, o, v);
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_correct_fast(double* __restrict__ P, Lvl L,
                                                      const double* __restrict__ Pc, Lvl Lc,
                                                      BcSpec bc) {
    int bb[3];
    if (!tile_coords<D>(L, bb)) return;
    correct_pt<D>(P, L, Pc, Lc, bc, bb);
}

// residual into R (edge fields: input of the tangential restriction)
template <int D, int EA>
__device__ __forceinline__ void residual_pt(const double* __restrict__ P,
                                            const double* __restrict__ F, double* __restrict__ R,
                                            const Lvl& L, const int* bb) {
    const long o0 = at<D>(L, 0, bb[0], bb[1], bb[2]);
#pragma unroll
    for (int c = 0; c < (1 << D); ++c) {
        if (is_wall<D, EA>(L, c, bb)) continue;
        const long o = o0 + (long)c * L.cls;
        R[o] = sb(F[o], op_fast<D>(P, L, c, o));
    }
}

template <int D, int EA>
__global__ void __launch_bounds__(256) k_residual_fast(const double* __restrict__ P,
                                                       const double* __restrict__ F,
                                                       double* __restrict__ R, Lvl L) {
    int bb[3];
    if (!tile_coords<D>(L, bb)) return;
    residual_pt<D, EA>(P, F, R, L, bb);
}

// Outer residual sum of squares of a cell-centred level, structured like
// k_tau_fast: every load of the block (2^d centers, 2^d f, d*2^(d-1)
// across-face neighbours) is issued before any arithmetic, so a warp keeps
// ~3x more DRAM requests in flight than the per-class op_fast loop.  Same
// per-point arithmetic (op_fast order), same per-CTA fixed-order partials.
template <int D>
__global__ void __launch_bounds__(256) k_res_sumsq_cell(const double* __restrict__ P,
                                                        const double* __restrict__ F, Lvl L,
                                                        double* __restrict__ part, int chunk) {
    int bb[3];
    double acc = 0.0;
    const bool act = tile_coords<D>(L, bb);
    // each thread walks `chunk` consecutive blocks along axis 0 (fewer CTAs,
    // one CTA reduction per chunk)
    const int b0s = (bb[0] - 1) * chunk + 1;
    for (int i = 0; act && i < chunk && b0s + i <= L.B[0]; ++i) {
        bb[0] = b0s + i;
        constexpr int NC = 1 << D;
        const long o0 = at<D>(L, 0, bb[0], bb[1], bb[2]);
        double pc[NC], fv[NC], out[NC][D];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const long o = o0 + (long)c * L.cls;
            pc[c] = __ldg(P + o);
            fv[c] = __ldg(F + o);
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const int bit = 1 << (D - 1 - a);
                const long dcls = (long)((c ^ bit) - c) * L.cls;
                const long sa = bstride<D>(L, a);
                out[c][a] = (c & bit) ? __ldg(P + o + dcls - sa) : __ldg(P + o + dcls + sa);
            }
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            double ns = 0.0;
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const int bit = 1 << (D - 1 - a);
                const double inside = pc[c ^ bit];
                const double e = (c & bit) ? inside : out[c][a];
                const double w = (c & bit) ? out[c][a] : inside;
                ns = a == 0 ? ad(e, w) : ad(ad(ns, e), w);
            }
            const double lap = ml(sb(ns, ml(D == 3 ? 6.0 : 4.0, pc[c])), L.inv_h2);
            const double r = sb(fv[c], sb(ml(L.a, pc[c]), ml(L.b, lap)));
            acc = ad(acc, ml(r, r));
        }
    }
    // fixed-order tree over the CTA (block sizes are powers of two <= 256)
    __shared__ double red[256];
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int nt = blockDim.x * blockDim.y * blockDim.z;
    red[tid] = acc;
    __syncthreads();
    for (int s = nt >> 1; s > 0; s >>= 1) {
        if (tid < s) red[tid] = ad(red[tid], red[tid + s]);
        __syncthreads();
    }
    if (tid == 0) part[blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)] = red[0];
}

// outer residual sum of squares: per-CTA fixed-order partials
template <int D, int EA>
__global__ void __launch_bounds__(256) k_res_sumsq_fast(const double* __restrict__ P,
                                                        const double* __restrict__ F, Lvl L,
                                                        double* __restrict__ part) {
    int bb[3];
    double acc = 0.0;
    if (tile_coords<D>(L, bb)) {
        const long o0 = at<D>(L, 0, bb[0], bb[1], bb[2]);
#pragma unroll
        for (int c = 0; c < (1 << D); ++c) {
            if (is_wall<D, EA>(L, c, bb)) continue;
            const long o = o0 + (long)c * L.cls;
            const double r = sb(F[o], op_fast<D>(P, L, c, o));
            acc = ad(acc, ml(r, r));
        }
    }
    // fixed-order tree over the CTA (block sizes are powers of two <= 256)
    __shared__ double red[256];
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int nt = blockDim.x * blockDim.y * blockDim.z;
    red[tid] = acc;
    __syncthreads();
    for (int s = nt >> 1; s > 0; s >>= 1) {
        if (tid < s) red[tid] = ad(red[tid], red[tid + s]);
        __syncthreads();
    }
    if (tid == 0) part[blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)] = red[0];
}

