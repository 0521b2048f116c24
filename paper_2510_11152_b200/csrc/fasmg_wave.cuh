// fasmg_wave.cuh -- temporally blocked X-MCGS smoothing for large 3D levels
// (included by fasmg_engine.cu inside namespace fasmg, after
// fasmg_stencil.cuh).
//
// One persistent launch runs T consecutive half-sweeps of one level (the 8
// half-sweeps of a smoothing stage at s=2, 'ff': PKG/fas.py:98,124 calling
// PKG/smoothers.py:136-153 twice) as a wavefront along block axis 0.
//
// Work item = (half-sweep t, block plane b0, 32x8 tile of (b2, b1) blocks).
// A half-sweep's 7-point stencil reaches one block either side along every
// axis, so item (t, b, tile in tile row r) may run once half-sweep t-1 has
// finished tile rows r-1..r+1 of planes b-1..b+1 (its inputs are final, and
// every earlier reader of the classes it overwrites is done -- transitively
// this covers all earlier half-sweeps).  A tile row spans the whole b2
// extent, which covers the in-plane periodic wrap along b2; with a periodic
// b1 axis the first and last tile rows are neighbours (the b1 ghost row of
// one is written by the other).  A periodic axis 0 would couple the first
// and last planes and is not run by this kernel.
//
// Every point is updated with exactly the arithmetic and the ghost-pad
// maintenance of k_sweep_smem / k_sweep_fast, and in the same dependency
// order as the reference's color sequence, so results are bitwise equal.
//
// CTA = 8 consumer warps (one thread per block of the tile; the 4 classes
// of the half-sweep's color) + 1 producer warp + 1 signaler warp.  The producer takes
// tickets, waits for the item's dependency counters (ld.acquire.gpu), and
// issues TMA box loads into a 4-stage shared-memory ring (mbarrier
// complete_tx): per item the 4 opposite-parity classes at plane b0 with the
// in-plane halo the stencil needs (36 x 9: a TMA box must start on a 16-byte
// boundary -- an odd fp64 start coordinate is an illegal instruction on
// B200 -- so the column halo is widened to x0-2..x0+33), each opposite class's one
// axis-0 neighbor plane (32 x 8), and f of the 4 updated classes (32 x 8).
// TMA reads go to L2 (never a stale L1 line).  Consumers compute, store p
// (+ ghost pads) with plain stores and arrive (non-blocking) on the stage's
// named barrier; the signaler warp waits there, fences the stores to gpu
// scope, bumps the (t, b0) completion counter and frees the stage.
#pragma once

// (included inside namespace fasmg; <cuda.h> for CUtensorMap is included by
// fasmg_engine.cu at file scope)

namespace wave {
constexpr int TX = 32, TY = 8;            // tile of (b2, b1) blocks
constexpr int HX = TX + 4, HY = TY + 1;   // halo box (cols x0-2..x0+TX+1, 9 rows)
constexpr int HBOX = 336;                 // doubles per halo slot (324 -> 128 B multiple)
constexpr int IBOX = TX * TY;             // interior box
constexpr int STAGE_D = 4 * HBOX + 8 * IBOX;
constexpr int NST = 4;                    // ring stages (named barriers 1..NST)
constexpr int NCONS = TX * TY;            // consumer threads
constexpr int NTHR = NCONS + 64;          // + producer warp + signaler warp
constexpr unsigned TX_BYTES = 4u * HX * HY * 8u + 8u * IBOX * 8u;
constexpr size_t SMEM = (size_t)NST * STAGE_D * 8 + NST * 16 + 2 * NST * 8;
}  // namespace wave

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load4(void* dst, const CUtensorMap* map,
                                          unsigned long long* bar, int c0, int c1, int c2,
                                          int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"((unsigned long long)map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

struct WaveArgs {
    double* P;
    unsigned* flags;   // [T][B0+2][nty] per-tile-row completion counters (zeroed)
    unsigned* ticket;  // global ticket counter (zeroed before launch)
    int T;             // half-sweeps in this launch
    int lag;           // planes between consecutive half-sweeps in ticket order (1 or 2)
    unsigned odd;      // bit t: half-sweep t updates the odd-sum classes (0x96)
    int ntx, nty;      // tiles per plane along b2, b1
    int ng, K;         // tile groups per (t, plane), tiles per group
    int gpr;           // groups per tile row (a group never spans rows)
    int cyc1;          // axis 1 periodic: tile rows 0 and nty-1 are neighbours
    long long ngroups; // total tickets
    unsigned long long* trace;  // debug: 6 globaltimer stamps per item, or null
};

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// opposite classes of a color mask in ascending order -> slot index
template <unsigned OPP>
__device__ __forceinline__ constexpr int oslot(int k) {
    int n = 0;
    for (int t = 0; t < k; ++t) n += (OPP >> t) & 1u;
    return n;
}

// consumer side of one item for color mask M (0x96 or 0x69)
template <int EA, unsigned M>
__device__ __forceinline__ void wave_item(const double* __restrict__ S, const Lvl& L,
                                          const BcSpec& bc, double* __restrict__ P, int b0,
                                          int x0, int y0, int tx, int ty) {
    using namespace wave;
    constexpr unsigned OPP = M ^ 0xFFu;
    const double* H = S;                     // 4 halo boxes (opposite classes, plane b0)
    const double* X = S + 4 * HBOX;          // 4 axis-0 neighbor planes
    const double* Fb = S + 4 * HBOX + 4 * IBOX;  // f of the 4 updated classes
    double nv[8];
    int j = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        if (!((M >> c) & 1u)) continue;
        const int k0 = c ^ 4, k1 = c ^ 2, k2 = c ^ 1;
        // row of b1 in class k's halo box (start row y0 if q1(k) else y0-1)
        const int r0 = (k0 & 2) ? ty : ty + 1;
        const int r2 = (k2 & 2) ? ty : ty + 1;
        const double* h0 = H + oslot<OPP>(k0) * HBOX;
        const double* h1 = H + oslot<OPP>(k1) * HBOX;
        const double* h2 = H + oslot<OPP>(k2) * HBOX;
        const double cen0 = h0[r0 * HX + tx + 2];
        const double ext0 = X[oslot<OPP>(k0) * IBOX + ty * TX + tx];
        const double e0 = (c & 4) ? cen0 : ext0;
        const double w0 = (c & 4) ? ext0 : cen0;
        const double e1 = h1[(ty + 1) * HX + tx + 2];
        const double w1 = h1[ty * HX + tx + 2];
        const double e2 = (c & 1) ? h2[r2 * HX + tx + 2] : h2[r2 * HX + tx + 3];
        const double w2 = (c & 1) ? h2[r2 * HX + tx + 1] : h2[r2 * HX + tx + 2];
        // ((((E+W)+N)+S)+T)+B  (KER/numpy_backend.py:62)
        const double ns = ad(ad(ad(ad(ad(e0, w0), e1), w1), e2), w2);
        nv[c] = ad(ml(L.h2, Fb[j * IBOX + ty * TX + tx]), ml(L.b, ns));
        ++j;
    }
#pragma unroll
    for (int c = 0; c < 8; ++c)
        if ((M >> c) & 1u) nv[c] = dv(nv[c], L.denom);
    int bb[3] = {b0, y0 + ty, x0 + tx};
    const bool bnd = on_boundary<3>(L, bb);
    const long pl = at<3>(L, 0, bb[0], bb[1], bb[2]);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        if (!((M >> c) & 1u)) continue;
        if (is_wall<3, EA>(L, c, bb)) continue;
        const long o = pl + (long)c * L.cls;
        P[o] = nv[c];
        if (bnd) write_pads<3, EA>(P, L, bc, c, bb, o, nv[c]);
    }
}

template <int EA>
__global__ void __launch_bounds__(wave::NTHR, 2)
    k_smooth_wave(const __grid_constant__ CUtensorMap mapH, const __grid_constant__ CUtensorMap mapI,
                  const __grid_constant__ CUtensorMap mapF, Lvl L, BcSpec bc, WaveArgs A) {
    using namespace wave;
    extern __shared__ __align__(128) double sm[];
    int4* desc = (int4*)(sm + NST * STAGE_D);
    unsigned long long* full = (unsigned long long*)(desc + NST);
    unsigned long long* empty = full + NST;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int B0 = L.B[0];
    const int pstride = B0 + 2;
    const int ntiles = A.ntx * A.nty;

    if (tid >= NCONS + 32) {  // ------------- signaler warp
        // Publishes each finished item: waits (named barrier 1+stage) for the
        // consumers' stores, fences them to gpu scope, bumps the item's
        // completion counter and frees the ring stage -- so the consumers
        // never stall on the fence.
        int stage = 0;
        for (;;) {
            asm volatile("bar.sync %0, %1;" ::"r"(1 + stage), "n"(NCONS + 32) : "memory");
            const int4 d = desc[stage];
            if (d.x < 0) break;
            if (tid == NCONS + 32) {
                // the stage's shared memory is consumed: recycle it first,
                // then publish the item's global stores
                mbar_arrive(&empty[stage]);
                const int row = d.z / A.ntx;
                __threadfence();
                atomicAdd(A.flags + ((long)d.x * pstride + d.y) * A.nty + row, 1u);
                if (A.trace) A.trace[6 * (((long)d.x * B0 + (d.y - 1)) * ntiles + d.z) + 5] = gtime();
            }
            __syncwarp();
            if (++stage == NST) stage = 0;
        }
        return;
    }
    if (tid >= NCONS) {  // ---------------- producer warp (lane 0)
        if (tid != NCONS) return;
        int stage = 0;
        unsigned ph = 1;  // empty barriers start "released"
        const long long gpw = (long long)A.T * A.ng;
        long long g = (long long)atomicAdd(A.ticket, 1u);
        while (g < A.ngroups) {
            const long long gn = (long long)atomicAdd(A.ticket, 1u);  // next ticket, in flight
            const int w = (int)(g / gpw);
            const int r = (int)(g - (long long)w * gpw);
            const int t = r / A.ng, grp = r - t * A.ng;
            const int b = w + 1 - A.lag * t;
            g = gn;
            if (b < 1 || b > B0) continue;
            const unsigned long long tp0 = A.trace ? gtime() : 0ull;
            const int row = grp / A.gpr;  // tile row of this group
            if (t > 0) {
                // tile rows row-1..row+1 of planes b-1..b+1 of half-sweep t-1
                const int lo = max(1, b - 1), hi = min(B0, b + 1);
                for (;;) {
                    unsigned m = 0xFFFFFFFFu;
                    for (int q = lo; q <= hi; ++q) {
                        const unsigned* fl = A.flags + ((long)(t - 1) * pstride + q) * A.nty;
                        for (int dr = -1; dr <= 1; ++dr) {
                            int rr = row + dr;
                            if (A.cyc1) rr = (rr + A.nty) % A.nty;  // periodic b1 wrap
                            else if (rr < 0 || rr >= A.nty) continue;
                            m = min(m, ld_acquire(fl + rr));
                        }
                    }
                    if (m >= (unsigned)A.ntx) break;
                    __nanosleep(32);
                }
            }
            asm volatile("fence.proxy.async.global;" ::: "memory");
            const unsigned long long tp1 = A.trace ? gtime() : 0ull;
            const bool odd = (A.odd >> t) & 1u;
            const unsigned Mk = odd ? 0x96u : 0x69u;
            const unsigned OPP = Mk ^ 0xFFu;
            const int c0 = (grp - row * A.gpr) * A.K;
            const int te = row * A.ntx + min(A.ntx, c0 + A.K);
            for (int tile = row * A.ntx + c0; tile < te; ++tile) {
                mbar_wait(&empty[stage], ph);
                desc[stage] = make_int4(t, b, tile, 0);
                double* S = sm + stage * STAGE_D;
                const int ty0 = tile / A.ntx, tx0 = tile - ty0 * A.ntx;
                const int x0 = tx0 * TX + 1, y0 = ty0 * TY + 1;
                mbar_expect_tx(&full[stage], TX_BYTES);
                int n = 0, j = 0;
                for (int k = 0; k < 8; ++k) {
                    if ((OPP >> k) & 1u) {
                        tma_load4(S + n * HBOX, &mapH, &full[stage], OFF + x0 - 2,
                                  (k & 2) ? y0 : y0 - 1, b, k);
                        tma_load4(S + 4 * HBOX + n * IBOX, &mapI, &full[stage], OFF + x0, y0,
                                  (k & 4) ? b + 1 : b - 1, k);
                        ++n;
                    } else {
                        tma_load4(S + 4 * HBOX + 4 * IBOX + j * IBOX, &mapF, &full[stage],
                                  OFF + x0, y0, b, k);
                        ++j;
                    }
                }
                if (A.trace) {
                    unsigned long long* tr = A.trace + 6 * (((long)t * B0 + (b - 1)) * ntiles + tile);
                    tr[0] = tp0;
                    tr[1] = tp1;
                    tr[2] = gtime();
                }
                if (++stage == NST) { stage = 0; ph ^= 1u; }
            }
        }
        // sentinel: tell the consumers (and through them the signaler) to stop
        mbar_wait(&empty[stage], ph);
        desc[stage] = make_int4(-1, 0, 0, 0);
        mbar_arrive(&full[stage]);
        return;
    }

    // ------------------------------------ consumers (8 warps)
    const int tx = tid % TX, ty = tid / TX;
    int stage = 0;
    unsigned ph = 0;
    for (;;) {
        mbar_wait(&full[stage], ph);
        const int4 d = desc[stage];
        if (d.x >= 0) {
            const int t = d.x, b = d.y, tile = d.z;
            unsigned long long* tr =
                A.trace ? A.trace + 6 * (((long)t * B0 + (b - 1)) * ntiles + tile) : nullptr;
            if (tr && tid == 0) tr[3] = gtime();
            const int ty0 = tile / A.ntx, tx0 = tile - ty0 * A.ntx;
            const int x0 = tx0 * TX + 1, y0 = ty0 * TY + 1;
            const double* S = sm + stage * STAGE_D;
            if ((A.odd >> t) & 1u) wave_item<EA, 0x96u>(S, L, bc, A.P, b, x0, y0, tx, ty);
            else wave_item<EA, 0x69u>(S, L, bc, A.P, b, x0, y0, tx, ty);
            if (tr && tid == 0) tr[4] = gtime();
        }
        // hand the item to the signaler without waiting
        asm volatile("bar.arrive %0, %1;" ::"r"(1 + stage), "n"(NCONS + 32) : "memory");
        if (d.x < 0) break;
        if (++stage == NST) { stage = 0; ph ^= 1u; }
    }
}


// ---------------------------------------------------------------------------
// 2.5D marching half-sweep with TMA plane loads (3D, large levels).
// Same schedule as k_sweep_smem -- a CTA owns a 32 (b2) x 8 (b1) tile of
// block columns and marches a chunk of planes along b0, keeping for every
// opposite-parity class a 3-plane ring (the two window planes of the
// current step + the one being prefetched) -- but each plane tile of a
// class is ONE TMA box (36 x 10 doubles: the tile with its in-plane halo,
// starting on a 16-byte boundary) and f of the 4 updated classes comes in
// as four 32 x 8 boxes, all completing on one mbarrier per step.  One
// thread issues 8 bulk copies per step instead of every thread issuing
// ~6 cp.async of 8 bytes, which took the issue slots of the 8-byte version.
// Arithmetic and pad maintenance are those of k_sweep_fast.
namespace tsw {
constexpr int TX = 32, TY = 8, HX = TX + 4, HY = TY + 2;
constexpr int HB = 384;        // doubles per halo box slot (360 -> 128 B multiple)
constexpr int FB = TX * TY;    // f box
constexpr int RING = 3;
constexpr unsigned HBYTES = HX * HY * 8u, FBYTES = FB * 8u;
constexpr int CX = TX + 2, CY = TY + 2, CB = CX * CY;  // corr tile (block ring)
constexpr int CRING = 4;
constexpr size_t SMEM = (size_t)(4 * RING * HB + 2 * 4 * FB) * 8 + 2 * 8;
constexpr size_t SMEM_CORR = SMEM + (size_t)CRING * CB * 8;
}  // namespace tsw

// CORR: this is the FIRST post-smoothing half-sweep of the level and also
// applies the coarse correction (PKG/fas.py:119-124) on the fly -- the
// prolongation+correction fused into the first post-smoothing color.  The
// correction of fine block b is corr = p_c - pinit at its coarse cell (pinit
// = R(p) stored by the tau pass, bitwise what the reference stores).  Every
// opposite-color (B) neighbour is read as B + corr(its block); a boundary
// point's own ghost is rebuilt from its corrected value (the stored ghost
// predates the correction); the tile's B values stay uncorrected in memory
// -- the next half-sweep overwrites them without reading them -- but their
// ghost pads are written from the corrected values.  Because no CTA
// modifies a B value, neighbours read consistent data (no cross-CTA race).
// Requires: cell-centred, no periodic face, next half-sweep = the other color.
template <int EA, unsigned MASK, bool CORR = false>
__global__ void __launch_bounds__(256) k_sweep_tma(const __grid_constant__ CUtensorMap mapH,
                                                   const __grid_constant__ CUtensorMap mapF,
                                                   double* __restrict__ P, Lvl L, BcSpec bc,
                                                   int chunk, const double* __restrict__ Pc = nullptr,
                                                   const double* __restrict__ PIc = nullptr,
                                                   Lvl Lc = Lvl(), PeerHalo ph = PeerHalo()) {
    using namespace tsw;
    constexpr unsigned OPP = MASK ^ 0xFFu;
    extern __shared__ __align__(128) double sm[];
    double* opp = sm;                        // [4][RING][HB]
    double* fsm = sm + 4 * RING * HB;        // [2][4][FB]
    unsigned long long* bar = (unsigned long long*)(fsm + 2 * 4 * FB);
    double* csm = (double*)(bar + 2);        // (CORR) [CRING][CB] corrections, planes b0-1..b0+2
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
    const int x0 = blockIdx.x * TX + 1, y0 = blockIdx.y * TY + 1;
    const int b0s = 1 + blockIdx.z * chunk;
    const int b0e = min(L.B[0], b0s + chunk - 1);
    int bb[3];
    bb[2] = x0 + tx;
    bb[1] = y0 + ty;
    const bool active = bb[1] <= L.B[1] && bb[2] <= L.B[2];
    // (CORR) corrections p_c - pinit (PKG/fas.py:119) of a plane's corr tile:
    // block (y0-1+r, x0-1+q) at entry r*CX+q; thread tid covers entries tid
    // and tid+256.  corr_fetch only issues the loads (v: Pc, pinit pairs);
    // corr_store subtracts and stores -- a step later, so the latency hides.
    // The in-plane part of each entry's coarse offset (coarse class bits of
    // axes 1, 2 and the coarse blocks, coarse_of) is fixed for the launch:
    // computed once here, so a plane step adds only the axis-0 part.
    long cofs[2] = {0, 0};
    bool cok[2] = {false, false};
    if (CORR) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int e = tid + i * 256;
            const int b1 = y0 - 1 + e / CX, b2 = x0 - 1 + e % CX;
            cok[i] = e < CB && b1 >= 1 && b1 <= L.B[1] && b2 >= 1 && b2 <= L.B[2];
            cofs[i] = (long)(((b1 & 1) << 1) | (b2 & 1)) * Lc.cls + (long)((b1 + 1) >> 1) * Lc.s1 +
                      ((b2 + 1) >> 1) + OFF;
        }
    }
    auto corr_fetch = [&](int pl, double* v) {
        const int I0 = pl + L.off0;  // global fine block = coarse cell index
        const long po = (long)((I0 & 1) << 2) * Lc.cls + (long)(((I0 + 1) >> 1) - Lc.off0) * Lc.s0;
        const bool pok = pl >= 1 && pl <= L.B[0];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            v[2 * i] = v[2 * i + 1] = 0.0;
            if (pok && cok[i]) {
                v[2 * i] = __ldg(Pc + po + cofs[i]);
                v[2 * i + 1] = __ldg(PIc + po + cofs[i]);
            }
        }
    };
    static_assert((CRING & (CRING - 1)) == 0, "CRING must be a power of two");
    auto corr_store = [&](int pl, const double* v) {
        double* d = csm + (pl & (CRING - 1)) * CB;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int e = tid + i * 256;
            if (e < CB) d[e] = sb(v[2 * i], v[2 * i + 1]);
        }
    };
    if (CORR) {  // prologue: planes b0s-1, b0s, b0s+1 (all loads in flight at once)
        double v[3][4];
#pragma unroll
        for (int i = 0; i < 3; ++i) corr_fetch(b0s - 1 + i, v[i]);
#pragma unroll
        for (int i = 0; i < 3; ++i) corr_store(b0s - 1 + i, v[i]);
    }

    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // prologue: both window planes of every opposite class + f(b0s)
        unsigned long long* br = &bar[b0s & 1];
        mbar_expect_tx(br, 8 * HBYTES + 4 * FBYTES);
        int j = 0;
        for (int k = 0; k < 8; ++k) {
            if ((OPP >> k) & 1u) {
                const int lo = (k & 4) ? b0s : b0s - 1;
                for (int d = 0; d < 2; ++d)
                    tma_load4(opp + (oslot<OPP>(k) * RING + ((lo + d) % RING)) * HB, &mapH, br,
                              OFF + x0 - 2, y0 - 1, lo + d, k);
            } else {
                tma_load4(fsm + ((b0s & 1) * 4 + j) * FB, &mapF, br, OFF + x0, y0, b0s, k);
                ++j;
            }
        }
    }
    __syncthreads();
    const long col = at<3>(L, 0, 0, bb[1], bb[2]);

    for (int b0 = b0s; b0 <= b0e; ++b0) {
        if (tid == 0 && b0 < b0e) {  // prefetch the next step's new planes + f
            unsigned long long* br = &bar[(b0 + 1) & 1];
            mbar_expect_tx(br, 4 * HBYTES + 4 * FBYTES);
            int j = 0;
            for (int k = 0; k < 8; ++k) {
                if ((OPP >> k) & 1u) {
                    const int nxt = ((k & 4) ? b0 : b0 - 1) + 2;
                    tma_load4(opp + (oslot<OPP>(k) * RING + (nxt % RING)) * HB, &mapH, br,
                              OFF + x0 - 2, y0 - 1, nxt, k);
                } else {
                    tma_load4(fsm + (((b0 + 1) & 1) * 4 + j) * FB, &mapF, br, OFF + x0, y0,
                              b0 + 1, k);
                    ++j;
                }
            }
        }
        bb[0] = b0;
        const long pl = col + (long)b0 * L.s0;
        const int Bn[3] = {L.G0, L.B[1], L.B[2]};
        // (CORR) prefetch the corrections of plane b0+2 (stored at the end of
        // the step); this step's come from the shared ring
        double cpre[4] = {0.0, 0.0, 0.0, 0.0};
        if (CORR) corr_fetch(b0 + 2, cpre);
        double c_own = 0.0, cW[3] = {0.0, 0.0, 0.0}, cE[3] = {0.0, 0.0, 0.0};
        double araw[8];
        if (CORR && active) {
            const int cc0 = (ty + 1) * CX + tx + 1;
            const double* cp = csm + (b0 & (CRING - 1)) * CB;
            c_own = cp[cc0];
            cW[0] = csm[((b0 - 1) & (CRING - 1)) * CB + cc0];
            cE[0] = csm[((b0 + 1) & (CRING - 1)) * CB + cc0];
            cW[1] = cp[cc0 - CX];
            cE[1] = cp[cc0 + CX];
            cW[2] = cp[cc0 - 1];
            cE[2] = cp[cc0 + 1];
            // a point's own value is only needed for its ghost (boundary)
            if (on_boundary<3>(L, bb)) {
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    if ((MASK >> c) & 1u) araw[c] = __ldg(P + pl + (long)c * L.cls);
            } else {
#pragma unroll
                for (int c = 0; c < 8; ++c) araw[c] = 0.0;
            }
        }
        mbar_wait(&bar[b0 & 1], ((b0 - b0s) >> 1) & 1);
        if (active) {
            const int ci = (ty + 1) * HX + tx + 2;  // tile centre in a halo box
            const bool bnd = on_boundary<3>(L, bb);
            double nv[8];
            int j = 0;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                if (!((MASK >> c) & 1u)) continue;
                const int k0 = c ^ 4, k1 = c ^ 2, k2 = c ^ 1;
                const int lo0 = (k0 & 4) ? b0 : b0 - 1;
                const double* w0 = opp + oslot<OPP>(k0) * RING * HB;
                const double* wy = opp + (oslot<OPP>(k1) * RING + (b0 % RING)) * HB;
                const double* wz = opp + (oslot<OPP>(k2) * RING + (b0 % RING)) * HB;
                const bool q0 = (c & 4) != 0, q1 = (c & 2) != 0, q2 = (c & 1) != 0;
                double e0 = w0[((lo0 + 1) % RING) * HB + ci], w0v = w0[(lo0 % RING) * HB + ci];
                double e1 = wy[ci + (q1 ? 0 : HX)], w1 = wy[ci - (q1 ? HX : 0)];
                double e2 = wz[ci + (q2 ? 0 : 1)], w2 = wz[ci - (q2 ? 1 : 0)];
                if (CORR) {
                    // inside the block: own correction; across a face: the
                    // neighbour block's ...
                    if (q0) { e0 = ad(e0, c_own); w0v = ad(w0v, cW[0]); }
                    else { w0v = ad(w0v, c_own); e0 = ad(e0, cE[0]); }
                    if (q1) { e1 = ad(e1, c_own); w1 = ad(w1, cW[1]); }
                    else { w1 = ad(w1, c_own); e1 = ad(e1, cE[1]); }
                    if (q2) { e2 = ad(e2, c_own); w2 = ad(w2, cW[2]); }
                    else { w2 = ad(w2, c_own); e2 = ad(e2, cE[2]); }
                    if (bnd) {  // ... or, across a domain face, the own ghost
                        const double ac = ad(araw[c], c_own);  // corrected value of this point
                        auto gh = [&](int a, int sd) {
                            return bc.kind[a][sd] == BC_DIRICHLET ? sb(ml(2.0, bc.val[a][sd]), ac)
                                                                  : ac;
                        };
                        const int g0 = gb0(L, bb);
                        if (q0) { if (g0 == 1) w0v = gh(0, 0); }
                        else if (g0 == Bn[0]) e0 = gh(0, 1);
                        if (q1) { if (bb[1] == 1) w1 = gh(1, 0); }
                        else if (bb[1] == Bn[1]) e1 = gh(1, 1);
                        if (q2) { if (bb[2] == 1) w2 = gh(2, 0); }
                        else if (bb[2] == Bn[2]) e2 = gh(2, 1);
                    }
                }
                // ((((E+W)+N)+S)+T)+B  (KER/numpy_backend.py:62)
                double ns = ad(e0, w0v);
                ns = ad(ad(ns, e1), w1);
                ns = ad(ad(ns, e2), w2);
                nv[c] = ad(ml(L.h2, fsm[((b0 & 1) * 4 + j) * FB + tid]), ml(L.b, ns));
                ++j;
            }
#pragma unroll
            for (int c = 0; c < 8; ++c)
                if ((MASK >> c) & 1u) nv[c] = dv(nv[c], L.denom);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                if (!((MASK >> c) & 1u)) continue;
                if (is_wall<3, EA>(L, c, bb)) continue;
                const long o = pl + (long)c * L.cls;
                P[o] = nv[c];
                if (bnd) write_pads<3, EA>(P, L, bc, c, bb, o, nv[c]);
                push_halo<3>(ph, L, c, bb, nv[c]);
            }
            if (CORR && bnd) {  // ghosts of the (uncorrected in memory) B points
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (!((OPP >> k) & 1u)) continue;
                    const double braw = opp[(oslot<OPP>(k) * RING + (b0 % RING)) * HB + ci];
                    write_pads<3, EA>(P, L, bc, k, bb, pl + (long)k * L.cls, ad(braw, c_own));
                }
            }
        }
        if (CORR) corr_store(b0 + 2, cpre);  // ring slot of plane b0-2: unused from now on
        __syncthreads();  // the next prefetch overwrites this step's oldest slots
    }
}

// ---------------------------------------------------------------------------
// Residual of a cell-centred level on the same TMA march (k_sweep_tma's
// tile/chunk geometry): per plane step one thread issues, for each of the
// 8 classes, the plane-b0 tile with its in-plane halo (36 x 10) by TMA,
// double-buffered on two mbarriers; f and the one axis-0 neighbour each
// class needs (b0+1 for q0=1 classes, b0-1 for q0=0 -- L2 hits, that plane
// is a neighbouring step's TMA box) are read straight from global, issued
// before the barrier wait.  40 KB of shared memory per CTA: 4 CTAs per SM.  MODE 0 accumulates sum(r^2) (outer norm, PKG/fas.py:149-151;
// per-CTA fixed-order partials); MODE 1 restricts r and p into the coarse
// level (tau pass, PKG/fas.py:99-107) with tau_pt's exact arithmetic.
namespace rsw {
constexpr int TX = 32, TY = 8, HX = TX + 4, HB = 384, IB = TX * TY;
constexpr size_t SLOT = (size_t)8 * HB;  // halo boxes (axis-0 neighbours: direct loads)
constexpr size_t SMEM = 2 * SLOT * 8 + 2 * 8;
constexpr unsigned TXB = 8u * HX * (TY + 2) * 8u;
}  // namespace rsw

template <int MODE, int EA = -1>
__global__ void __launch_bounds__(256) k_resid_tma(const __grid_constant__ CUtensorMap mapH,
                                                   const double* __restrict__ P,
                                                   const double* __restrict__ F, Lvl L,
                                                   BcSpec bc, int chunk,
                                                   double* __restrict__ part,
                                                   double* __restrict__ Pc,
                                                   double* __restrict__ Fc, Lvl Lc,
                                                   double* __restrict__ PIc) {
    using namespace rsw;
    extern __shared__ __align__(128) double sm[];
    unsigned long long* bar = (unsigned long long*)(sm + 2 * SLOT);
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
    const int x0 = blockIdx.x * TX + 1, y0 = blockIdx.y * TY + 1;
    const int b0s = 1 + blockIdx.z * chunk;
    const int b0e = min(L.B[0], b0s + chunk - 1);
    auto issue = [&](int b0, int s) {
        double* S = sm + s * SLOT;
        mbar_expect_tx(&bar[s], TXB);
        for (int k = 0; k < 8; ++k)
            tma_load4(S + k * HB, &mapH, &bar[s], OFF + x0 - 2, y0 - 1, b0, k);
    };
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        issue(b0s, 0);
    }
    __syncthreads();
    const int b1 = y0 + ty, b2 = x0 + tx;
    const bool active = b1 <= L.B[1] && b2 <= L.B[2];
    const int ci = (ty + 1) * HX + tx + 2;  // tile centre in a halo box
    double acc = 0.0;
    for (int b0 = b0s; b0 <= b0e; ++b0) {
        const int s = (b0 - b0s) & 1;
        if (tid == 0 && b0 < b0e) issue(b0 + 1, s ^ 1);
        // f and the axis-0 neighbour plane of every class straight from global
        // (coalesced rows, L2-resident), issued before the barrier wait
        double fv[8], nb0[8];
        if (active) {
            const long o = at<3>(L, 0, b0, b1, b2);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                fv[c] = __ldg(F + o + (long)c * L.cls);
                nb0[c] = P[o + (long)c * L.cls + ((c & 4) ? L.s0 : -L.s0)];
            }
        }
        mbar_wait(&bar[s], ((b0 - b0s) >> 1) & 1);
        const double* S = sm + s * SLOT;
        if (active) {
            double pc[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) pc[c] = S[c * HB + ci];
            double rp = 0.0, rr = 0.0;
#pragma unroll
            for (int c = 7; c >= 0; --c) {
                double ns = 0.0;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const int bit = 1 << (2 - a);
                    const bool qa = (c & bit) != 0;
                    const int k = c ^ bit;
                    const double inside = pc[k];
                    // across the block face: W of q=1, E of q=0
                    double out;
                    if (a == 0) out = nb0[k];
                    else if (a == 1) out = S[k * HB + ci + (qa ? -HX : HX)];
                    else out = S[k * HB + ci + (qa ? -1 : 1)];
                    const double e = qa ? inside : out;
                    const double w = qa ? out : inside;
                    ns = a == 0 ? ad(e, w) : ad(ad(ns, e), w);
                }
                const double lap = ml(sb(ns, ml(6.0, pc[c])), L.inv_h2);
                const double r = sb(fv[c], sb(ml(L.a, pc[c]), ml(L.b, lap)));
                if (MODE == 0) {
                    // edge fields: wall points are not unknowns (PKG/grid.py:199-208)
                    int bw[3] = {b0, b1, b2};
                    if (!is_wall<3, EA>(L, c, bw)) acc = ad(acc, ml(r, r));
                } else {
                    if (c == 7) { rp = pc[c]; rr = r; }
                    else { rp = ad(rp, pc[c]); rr = ad(rr, r); }
                }
            }
            if (MODE == 1) {
                int bb[3] = {b0, b1, b2}, cc = 0, cb[3] = {0, 0, 0};
                coarse_of<3>(L, Lc, bb, cc, cb);
                const long oc = at<3>(Lc, cc, cb[0], cb[1], cb[2]);
                const double pcv = ml(rp, 0.125);
                Pc[oc] = pcv;
                if (PIc) PIc[oc] = pcv;  // pinit, for the fused correction
                Fc[oc] = ml(rr, 0.125);
                if (on_boundary<3>(Lc, cb)) write_pads<3, -1>(Pc, Lc, bc, cc, cb, oc, pcv);
            }
        }
        __syncthreads();  // slot s is refilled by the next step's prefetch
    }
    if (MODE == 0) {
        double* red = sm;  // the ring is free now
        red[tid] = acc;
        __syncthreads();
        for (int s2 = 128; s2 > 0; s2 >>= 1) {
            if (tid < s2) red[tid] = ad(red[tid], red[tid + s2]);
            __syncthreads();
        }
        if (tid == 0) part[blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)] = red[0];
    }
}

// ---------------------------------------------------------------------------
// 2D half-sweep fed by TMA.  A CTA owns a 32 (b1) x 8 (b0) tile and walks
// `steps` consecutive tiles down axis 0; per step ONE thread issues the two
// opposite classes' tile + 1-block halo (36 x 10 box, 16-byte aligned start)
// and f of the two updated classes (32 x 8), double-buffered on two
// mbarriers so the next tile's loads overlap this tile's arithmetic.  Same
// per-point arithmetic / pad maintenance as sweep_pt<2>.
namespace tsw2 {
constexpr int TX = 32, TY = 8, HX = TX + 4, HY = TY + 2, HB = 384, FB = TX * TY;
constexpr size_t SLOT = 2 * HB + 2 * FB;
constexpr size_t SMEM = 2 * SLOT * 8 + 2 * 8;
constexpr unsigned TXB = 2u * HX * HY * 8u + 2u * FB * 8u;
}  // namespace tsw2

__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* map,
                                          unsigned long long* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"((unsigned long long)map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

template <int EA, unsigned MASK>
__global__ void __launch_bounds__(256) k_sweep_tma2d(const __grid_constant__ CUtensorMap mapH,
                                                     const __grid_constant__ CUtensorMap mapF,
                                                     double* __restrict__ P, Lvl L, BcSpec bc,
                                                     int steps, PeerHalo ph = PeerHalo()) {
    using namespace tsw2;
    constexpr unsigned OPP = MASK ^ 0xFu;
    extern __shared__ __align__(128) double sm[];
    unsigned long long* bar = (unsigned long long*)(sm + 2 * SLOT);
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
    const int x0 = blockIdx.x * TX + 1;
    const int r0 = 1 + blockIdx.y * steps * TY;  // first block row of this CTA
    const int nst = min(steps, (L.B[0] - r0 + TY) / TY);
    auto issue = [&](int st, int s) {
        double* S = sm + s * SLOT;
        const int y0 = r0 + st * TY;
        mbar_expect_tx(&bar[s], TXB);
        int n = 0, j = 0;
        for (int k = 0; k < 4; ++k) {
            if ((OPP >> k) & 1u) {
                tma_load3(S + n * HB, &mapH, &bar[s], OFF + x0 - 2, y0 - 1, k);
                ++n;
            } else {
                tma_load3(S + 2 * HB + j * FB, &mapF, &bar[s], OFF + x0, y0, k);
                ++j;
            }
        }
    };
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (nst > 0) issue(0, 0);
    }
    __syncthreads();
    const int ci = (ty + 1) * HX + tx + 2;
    for (int st = 0; st < nst; ++st) {
        const int s = st & 1;
        if (tid == 0 && st + 1 < nst) issue(st + 1, s ^ 1);
        mbar_wait(&bar[s], (st >> 1) & 1);
        const double* S = sm + s * SLOT;
        int bb[3] = {r0 + st * TY + ty, x0 + tx, 0};
        if (bb[0] <= L.B[0] && bb[1] <= L.B[1]) {
            double nv[4];
            int j = 0;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                if (!((MASK >> c) & 1u)) continue;
                const int k0 = c ^ 2, k1 = c ^ 1;
                const double* h0 = S + oslot<OPP>(k0) * HB;
                const double* h1 = S + oslot<OPP>(k1) * HB;
                const bool q0 = (c & 2) != 0, q1 = (c & 1) != 0;
                // ((E+W)+N)+S  (KER/numpy_backend.py:44)
                double ns = ad(h0[ci + (q0 ? 0 : HX)], h0[ci - (q0 ? HX : 0)]);
                ns = ad(ad(ns, h1[ci + (q1 ? 0 : 1)]), h1[ci - (q1 ? 1 : 0)]);
                nv[c] = ad(ml(L.h2, S[2 * HB + j * FB + tid]), ml(L.b, ns));
                ++j;
            }
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if ((MASK >> c) & 1u) nv[c] = dv(nv[c], L.denom);
            const bool bnd = on_boundary<2>(L, bb);
            const long pl = at<2>(L, 0, bb[0], bb[1], 0);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                if (!((MASK >> c) & 1u)) continue;
                if (is_wall<2, EA>(L, c, bb)) continue;
                const long o = pl + (long)c * L.cls;
                P[o] = nv[c];
                if (bnd) write_pads<2, EA>(P, L, bc, c, bb, o, nv[c]);
                push_halo<2>(ph, L, c, bb, nv[c]);
            }
        }
        __syncthreads();  // slot s is refilled by the next step's prefetch
    }
}
