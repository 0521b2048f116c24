// fasmg_wave.cuh -- TMA-fed marching kernels for large levels: the 3D
// X-MCGS half-sweep (k_sweep_tma, optionally with the coarse correction
// fused in), the residual march (k_resid_tma: tau pass and outer norm) and
// the 2D half-sweep (k_sweep_tma2d).  Included by fasmg_engine.cu inside
// namespace fasmg, after fasmg_stencil.cuh.
#pragma once

// (included inside namespace fasmg; <cuda.h> for CUtensorMap is included by
// fasmg_engine.cu at file scope)

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
    // the lanes of a warp can leave the spin at different polls: reconverge
    // before the caller's next block barrier.  Every caller waits with all
    // 32 lanes.
    __syncwarp();
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

// opposite classes of a color mask in ascending order -> slot index
template <unsigned OPP>
__device__ __forceinline__ constexpr int oslot(int k) {
    int n = 0;
    for (int t = 0; t < k; ++t) n += (OPP >> t) & 1u;
    return n;
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
// edge CORR sweep: f from global (1) or TMA f boxes (0)
#ifndef EC_FG
#define EC_FG 0
#endif
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
// (edge CORR) coarse Corr tiles: coarse indices y0-2..y0+9 x x0-3..x0+34
// of one coarse plane per slot, ERING planes (c0-1..c0+3 of step c0)
constexpr int ECX = TX + 6, ECY = TY + 4, ECP = ECX * ECY, ERING = 5;
// (f read straight from global in that variant: no f boxes)
constexpr size_t SMEM_ECORR = SMEM - (EC_FG ? (size_t)2 * 4 * FB * 8 : 0) + (size_t)ERING * ECP * 8;
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
//
// Edge fields (EA >= 0) with CORR: the correction is the edge prolongation
// (KER/numpy_backend.py:194-224, correct_edge_pt) of the coarse Corr array
// (Pc = Corr: p_c - pinit with the homogenized ghost chain, k_corr_edge_*),
// which varies inside a block, so it is applied where the data already is:
// each opposite-class halo box is corrected IN SHARED MEMORY once, when its
// plane arrives, from a ring of coarse Corr tiles (one coarse plane per
// step: fine block b sits on coarse index b along every axis).  The sweep
// arithmetic is then unchanged; across a domain face a boundary point's
// neighbour is its own ghost / wall rebuilt from its corrected value
// (write_pads' rules), and the B points' ghosts are written from the
// corrected box values.
#define EC_BOUND ((CORR && EA >= 0) ? 3 : 0)
template <int EA, unsigned MASK, bool CORR = false>
__global__ void __launch_bounds__(256, EC_BOUND) k_sweep_tma(const __grid_constant__ CUtensorMap mapH,
                                                   const __grid_constant__ CUtensorMap mapF,
                                                   double* __restrict__ P, Lvl L, BcSpec bc,
                                                   int chunk, const double* __restrict__ Pc = nullptr,
                                                   const double* __restrict__ PIc = nullptr,
                                                   Lvl Lc = Lvl(), PeerHalo ph = PeerHalo(),
                                                   const double* __restrict__ Fg = nullptr) {
    using namespace tsw;
    constexpr unsigned OPP = MASK ^ 0xFFu;
    constexpr bool CC = CORR && EA < 0;   // cell: per-block constant correction
    constexpr bool EC = CORR && EA >= 0;  // edge: prolongation, boxes corrected in smem
    constexpr bool FG = EC && EC_FG;      // f read from global (Fg), not TMA boxes
    extern __shared__ __align__(128) double sm[];
    double* opp = sm;                        // [4][RING][HB]
    double* fsm = sm + 4 * RING * HB;        // [2][4][FB] (not FG)
    unsigned long long* bar = (unsigned long long*)(fsm + (FG ? 0 : 2 * 4 * FB));
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
    if (CC) {
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
    if (CC) {  // prologue: planes b0s-1, b0s, b0s+1 (all loads in flight at once)
        double v[3][4];
#pragma unroll
        for (int i = 0; i < 3; ++i) corr_fetch(b0s - 1 + i, v[i]);
#pragma unroll
        for (int i = 0; i < 3; ++i) corr_store(b0s - 1 + i, v[i]);
    }
    // (EC) coarse Corr ring: entry w = (c1 - (y0-2)) * ECX + (c2 - (x0-3)) of
    // the slot of coarse plane c0; thread tid fetches entries tid, tid+256
    // (in-plane part of the blocked offset fixed for the launch).  Pc = Corr
    // (k_corr_edge_in / k_corr_edge_pads: forming p_c - pinit here instead
    // costs more in this instruction-bound kernel than the separate pass)
    double* cring = (double*)(bar + 2);
    int eofs[2] = {-1, -1};  // (32-bit, -1: outside the level; as cofs)
    if (EC) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int w = tid + i * 256;
            const int c1 = y0 - 2 + w / ECX, c2 = x0 - 3 + w % ECX;
            if (w < ECP && c1 >= 0 && c2 >= 0 && ((c1 + 1) >> 1) < Lc.E[1] &&
                ((c2 + 1) >> 1) < Lc.E[2])
                eofs[i] = (((c1 & 1) << 1) | (c2 & 1)) * (int)Lc.cls + ((c1 + 1) >> 1) * (int)Lc.s1 +
                          ((c2 + 1) >> 1) + OFF;
        }
    }
    auto ec_slot = [&](int c0) { return ((c0 + 2 * ERING) % ERING) * ECP; };
    auto ec_fetch = [&](int c0, double* v) {
        const int k0 = ((c0 + 1) >> 1) - Lc.off0;
        const bool ok0 = c0 >= 0 && k0 >= 0 && k0 < Lc.E[0];
        const int po = ((c0 & 1) << 2) * (int)Lc.cls + k0 * (int)Lc.s0;
#pragma unroll
        for (int i = 0; i < 2; ++i) v[i] = (ok0 && eofs[i] >= 0) ? __ldg(Pc + (po + eofs[i])) : 0.0;
    };
    auto ec_store = [&](int c0, const double* v) {
        double* d = cring + ec_slot(c0);
#pragma unroll
        for (int i = 0; i < 2; ++i)
            if (tid + i * 256 < ECP) d[tid + i * 256] = v[i];
    };
    // correct_edge_pt's prolongation of Corr for class c at the fine block
    // whose coarse neighbourhood starts at tile offset rc (coarse (b1-1,
    // b2-1)) in the slots sA, sB, sC of coarse planes p-1, p, p+1 (axes
    // permuted: edge axis P0 first)
    auto eprol = [&](int c, int sA, int sB, int sC, int rc) -> double {
        constexpr int P0 = EA < 0 ? 0 : EA, P1 = P0 == 0 ? 1 : 0, P2 = P0 == 2 ? 1 : 2;
        auto cv = [&](int di, int dj, int dk) {
            const int d0 = P0 == 0 ? di : dj;
            const int d1 = P0 == 0 ? dj : (P0 == 1 ? di : dk);
            const int d2 = P0 == 2 ? di : dk;
            return cring[(d0 == 0 ? sA : (d0 == 1 ? sB : sC)) + rc + d1 * ECX + d2];
        };
        const int qe = (c >> (2 - P0)) & 1, qj = (c >> (2 - P1)) & 1, qk = (c >> (2 - P2)) & 1;
        const int jd = qj ? 0 : 2, kd = qk ? 0 : 2;
        auto line = [&](int i) {
            const double tn = ml(ad(ml(3.0, cv(i, 1, 1)), cv(i, jd, 1)), 0.25);
            const double tf = ml(ad(ml(3.0, cv(i, 1, kd)), cv(i, jd, kd)), 0.25);
            return ml(ad(ml(3.0, tn), tf), 0.25);
        };
        return qe ? ml(ad(line(0), line(1)), 0.5) : line(1);
    };
    // the box entries this thread corrects (launch constants): entry w =
    // tid + 256 i of the 34 x 10 blocks y0-1..y0+8 x x0-1..x0+32 (what the
    // sweep reads): box offset, tile offset, and the mask of the classes to
    // correct there -- interior points only (no pad block, no edge-axis
    // wall), and on the halo ring only the classes a tile point reads (the
    // row above: q1 = 0, below: q1 = 1, left: q2 = 0, right: q2 = 1; the
    // corners: none)
    int eb[2] = {0, 0}, er[2] = {0, 0};
    unsigned em[2] = {0u, 0u};
    if (EC) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int w = tid + i * 256;
            const int j = w / (TX + 2), col = w - j * (TX + 2);
            const int b1 = y0 - 1 + j, b2 = x0 - 1 + col;
            unsigned m = 0xFFu;
            if (j == 0) m &= 0x33u;
            if (j == TY + 1) m &= 0xCCu;
            if (col == 0) m &= 0x55u;
            if (col == TX + 1) m &= 0xAAu;
            if ((j == 0 || j == TY + 1) && (col == 0 || col == TX + 1)) m = 0u;
            if (!(w < (TX + 2) * (TY + 2) && b1 >= 1 && b1 <= L.B[1] && b2 >= 1 && b2 <= L.B[2]))
                m = 0u;
            if (EA == 1 && b1 == L.B[1]) m &= 0xCCu;  // q1 = 0 classes: the wall
            if (EA == 2 && b2 == L.B[2]) m &= 0xAAu;  // q2 = 0 classes: the wall
            em[i] = m;
            eb[i] = j * HX + col + 1;
            er[i] = j * ECX + col + 1;
        }
    }
    // add the correction to the interior points of the (class k, plane p)
    // halo box (ring slot rs of the plane); sA..sC: slots of coarse planes
    // p-1..p+1
    auto ecorrect = [&](int k, int p, int rs, int sA, int sB, int sC) {
        if (p < 1 || p > L.B[0]) return;  // pad plane: boundary points rebuild it
        if (EA == 0 && !(k & 4) && p + L.off0 == L.G0) return;  // the wall plane
        double* box = opp + (oslot<OPP>(k) * RING + rs) * HB;
#pragma unroll
        for (int i = 0; i < 2; ++i)
            if ((em[i] >> k) & 1u) box[eb[i]] = ad(box[eb[i]], eprol(k, sA, sB, sC, er[i]));
    };
    if (EC) {  // prologue: coarse planes b0s-2 .. b0s+2
        double v[5][2];
#pragma unroll
        for (int i = 0; i < 5; ++i) ec_fetch(b0s - 2 + i, v[i]);
#pragma unroll
        for (int i = 0; i < 5; ++i) ec_store(b0s - 2 + i, v[i]);
    }

    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // prologue: both window planes of every opposite class + f(b0s)
        unsigned long long* br = &bar[b0s & 1];
        mbar_expect_tx(br, 8 * HBYTES + (FG ? 0 : 4 * FBYTES));
        int j = 0;
        for (int k = 0; k < 8; ++k) {
            if ((OPP >> k) & 1u) {
                const int lo = (k & 4) ? b0s : b0s - 1;
                for (int d = 0; d < 2; ++d)
                    tma_load4(opp + (oslot<OPP>(k) * RING + ((lo + d) % RING)) * HB, &mapH, br,
                              OFF + x0 - 2, y0 - 1, lo + d, k);
            } else if (!FG) {
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
            mbar_expect_tx(br, 4 * HBYTES + (FG ? 0 : 4 * FBYTES));
            int j = 0;
            for (int k = 0; k < 8; ++k) {
                if ((OPP >> k) & 1u) {
                    const int nxt = ((k & 4) ? b0 : b0 - 1) + 2;
                    tma_load4(opp + (oslot<OPP>(k) * RING + (nxt % RING)) * HB, &mapH, br,
                              OFF + x0 - 2, y0 - 1, nxt, k);
                } else if (!FG) {
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
        if (CC) corr_fetch(b0 + 2, cpre);
        double epre[2] = {0.0, 0.0};
        if (EC) ec_fetch(b0 + 3, epre);  // stored at the end of the step
        // (EC) ring slots of coarse planes b0-2 (esm), b0-1 (es0) .. b0+2 (es3)
        int esm = 0, es0 = 0, es1 = 0, es2 = 0, es3 = 0;
        // (EC) halo-box ring slots of planes b0-1, b0, b0+1
        const int r0 = b0 % RING, rm = r0 == 0 ? RING - 1 : r0 - 1, rp = r0 == RING - 1 ? 0 : r0 + 1;
        if (EC) {
            const int t = (b0 + 2 * ERING - 2) % ERING;
            auto sl = [&](int m) { return (t + m >= ERING ? t + m - ERING : t + m) * ECP; };
            esm = sl(0); es0 = sl(1); es1 = sl(2); es2 = sl(3); es3 = sl(4);
        }
        double c_own = 0.0, cW[3] = {0.0, 0.0, 0.0}, cE[3] = {0.0, 0.0, 0.0};
        double araw[8];
        if (CC && active) {
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
        double fv[4] = {0.0, 0.0, 0.0, 0.0};
        if (FG && active) {  // f of the updated classes (no f boxes in this variant)
            int j = 0;
#pragma unroll
            for (int c = 0; c < 8; ++c)
                if ((MASK >> c) & 1u) fv[j++] = __ldg(Fg + pl + (long)c * L.cls);
        }
        if (EC && active && on_boundary<3>(L, bb)) {  // own raw values: ghosts / walls
#pragma unroll
            for (int c = 0; c < 8; ++c)
                if ((MASK >> c) & 1u) araw[c] = __ldg(P + pl + (long)c * L.cls);
        }
        mbar_wait(&bar[b0 & 1], ((b0 - b0s) >> 1) & 1);
        if (EC) {  // correct the planes that arrived for this step
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (!((OPP >> k) & 1u)) continue;
                if (k & 4) {  // plane b0+1 (and b0 on the first step)
                    ecorrect(k, b0 + 1, rp, es1, es2, es3);
                    if (b0 == b0s) ecorrect(k, b0, r0, es0, es1, es2);
                } else {      // plane b0 (and b0-1 on the first step)
                    ecorrect(k, b0, r0, es0, es1, es2);
                    if (b0 == b0s) ecorrect(k, b0 - 1, rm, esm, es0, es1);
                }
            }
            __syncthreads();
        }
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
                if (CC) {
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
                if (EC && bnd) {  // across a domain face: own ghost / wall (write_pads)
                    const double ac =
                        ad(araw[c], eprol(c, es0, es1, es2,
                                          (ty + 1) * ECX + tx + 2));
                    auto gh = [&](int a, int sd, double raw) {
                        const int kd = bc.kind[a][sd];
                        if (a != EA) return kd == BC_DIRICHLET ? sb(ml(2.0, bc.val[a][sd]), ac) : ac;
                        return kd == BC_NEUMANN ? ac : raw;
                    };
                    // lo face: W of a q=1 point at g=1; hi face: E of a q=0
                    // point at g=B, or (edge axis) of the q=1 point at g=B
                    const int g0 = gb0(L, bb);
                    if (q0 && g0 == 1) w0v = gh(0, 0, w0v);
                    if ((EA == 0 ? q0 : !q0) && g0 == Bn[0]) e0 = gh(0, 1, e0);
                    if (q1 && bb[1] == 1) w1 = gh(1, 0, w1);
                    if ((EA == 1 ? q1 : !q1) && bb[1] == Bn[1]) e1 = gh(1, 1, e1);
                    if (q2 && bb[2] == 1) w2 = gh(2, 0, w2);
                    if ((EA == 2 ? q2 : !q2) && bb[2] == Bn[2]) e2 = gh(2, 1, e2);
                }
                // ((((E+W)+N)+S)+T)+B  (KER/numpy_backend.py:62)
                double ns = ad(e0, w0v);
                ns = ad(ad(ns, e1), w1);
                ns = ad(ad(ns, e2), w2);
                nv[c] = ad(ml(L.h2, FG ? fv[j] : fsm[((b0 & 1) * 4 + j) * FB + tid]), ml(L.b, ns));
                ++j;
            }
#pragma unroll
            for (int c = 0; c < 8; ++c)
                if ((MASK >> c) & 1u) nv[c] = dvr(nv[c], L.denom, L.rden);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                if (!((MASK >> c) & 1u)) continue;
                if (is_wall<3, EA>(L, c, bb)) continue;
                const long o = pl + (long)c * L.cls;
                P[o] = nv[c];
                if (bnd) write_pads<3, EA>(P, L, bc, c, bb, o, nv[c]);
                push_halo<3>(ph, L, c, bb, nv[c]);
            }
            if (CC && bnd) {  // ghosts of the (uncorrected in memory) B points
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (!((OPP >> k) & 1u)) continue;
                    const double braw = opp[(oslot<OPP>(k) * RING + (b0 % RING)) * HB + ci];
                    write_pads<3, EA>(P, L, bc, k, bb, pl + (long)k * L.cls, ad(braw, c_own));
                }
            }
            if (EC && bnd) {  // ghosts of the B points from their corrected (box) values
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (!((OPP >> k) & 1u) || is_wall<3, EA>(L, k, bb)) continue;
                    const double bv = opp[(oslot<OPP>(k) * RING + (b0 % RING)) * HB + ci];
                    write_pads<3, EA>(P, L, bc, k, bb, pl + (long)k * L.cls, bv);
                }
            }
        }
        if (CC) corr_store(b0 + 2, cpre);  // ring slot of plane b0-2: unused from now on
        if (EC) ec_store(b0 + 3, epre);    // slot of plane b0-2: unused from now on
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

// MODE 2 (cell fields): the outer norm of MODE 0 AND, from the same loaded
// values, the NEXT V-cycle's first pre-smoothing half-sweep of the classes
// in MX (speculative: the host decides afterwards whether that cycle runs).
// A half-sweep reads exactly what the residual reads -- the opposite
// classes around the point (box + axis-0 neighbour), f, in the same
// ((((E+W)+N)+S)+T)+B order -- so X_new = (h2*f + b*ns)/denom costs no extra
// load.  X_new goes to P2 (P keeps the state the norm describes), with the
// ghosts the next half-sweep reads: ghost(Y_old) into P2's X-class pads;
// ghost(X_new) into P's Y-class pads (read only by the third half-sweep;
// a stop before it rebuilds P's pads, fasmg_engine spec_cancel).  The only
// reader of a pad slot written here is the thread that writes it, and it
// read the slot first.
template <int MODE, int EA = -1, bool RESID_PF = false, unsigned MX = 0u>
__global__ void __launch_bounds__(256) k_resid_tma(const __grid_constant__ CUtensorMap mapH,
                                                   const double* __restrict__ P,
                                                   const double* __restrict__ F, Lvl L,
                                                   BcSpec bc, int chunk,
                                                   double* __restrict__ part,
                                                   double* __restrict__ Pc,
                                                   double* __restrict__ Fc, Lvl Lc,
                                                   double* __restrict__ PIc,
                                                   double* __restrict__ P2 = nullptr,
                                                   double* Pw = nullptr) {
    static_assert(MODE != 2 || (EA == -1 && MX != 0u), "MODE 2: cell fields, a class mask");
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
    // f and the axis-0 neighbour plane of every class straight from global
    // (coalesced rows, L2-resident), loaded one plane step AHEAD so their
    // latency hides behind the current plane's arithmetic (RESID_PF)
    double fv[8], nb0[8];
    auto load_tile = [&](int b0) {
        if (!active) return;
        const long o = at<3>(L, 0, b0, b1, b2);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            fv[c] = __ldg(F + o + (long)c * L.cls);
            nb0[c] = P[o + (long)c * L.cls + ((c & 4) ? L.s0 : -L.s0)];
        }
    };
    if (RESID_PF) load_tile(b0s);
    for (int b0 = b0s; b0 <= b0e; ++b0) {
        const int s = (b0 - b0s) & 1;
        if (tid == 0 && b0 < b0e) issue(b0 + 1, s ^ 1);
        if (!RESID_PF) load_tile(b0);  // issued before the barrier wait
        mbar_wait(&bar[s], ((b0 - b0s) >> 1) & 1);
        const double* S = sm + s * SLOT;
        if (active) {
            double pc[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) pc[c] = S[c * HB + ci];
            double rp = 0.0, rr = 0.0;
            double xn[8];  // (MODE 2) numerators of the speculative half-sweep
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
                if (MODE == 2 && ((MX >> c) & 1u)) xn[c] = ad(ml(L.h2, fv[c]), ml(L.b, ns));
                if (MODE == 0 || MODE == 2) {
                    // edge fields: wall points are not unknowns (PKG/grid.py:199-208)
                    int bw[3] = {b0, b1, b2};
                    if (!is_wall<3, EA>(L, c, bw)) acc = ad(acc, ml(r, r));
                } else {
                    if (c == 7) { rp = pc[c]; rr = r; }
                    else { rp = ad(rp, pc[c]); rr = ad(rr, r); }
                }
            }
            if (MODE == 2) {
                int bb[3] = {b0, b1, b2};
                const bool bnd = on_boundary<3>(L, bb);
                const long o = at<3>(L, 0, b0, b1, b2);
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    if ((MX >> c) & 1u) {
                        const double v = dvr(xn[c], L.denom, L.rden);
                        P2[o + (long)c * L.cls] = v;
                        if (bnd) write_pads<3, -1>(Pw, L, bc, c, bb, o + (long)c * L.cls, v);
                    } else if (bnd) {
                        write_pads<3, -1>(P2, L, bc, c, bb, o + (long)c * L.cls, pc[c]);
                    }
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
        if (RESID_PF && b0 < b0e) load_tile(b0 + 1);
        __syncthreads();  // slot s is refilled by the next step's prefetch
    }
    if (MODE == 0 || MODE == 2) {
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
// Edge-field (MAC face velocity) tau pass in ONE TMA march (3D): the
// residual r = f - A p, the (1,2,1)x(1,2,1)x(1/2) edge restriction of both r
// and p (KER/numpy_backend.py:162-191; PKG/fas.py:99-107) and the coarse
// outputs p_c, pinit = p_c and f_c = R(r) -- replacing k_residual_fast +
// k_pad_all2 + 2 x k_restrict_edge_fast + the pinit copy (the r array is
// never written).  k_coarse_src_fast then adds L_2h(p_c).
//
// Coarse point I (per axis) restricts fine block I: along the edge axis EA
// both classes (columns 2I-1, 2I), along a tangential axis t the classes of
// block I and the first class (bit 1, row 2I+1) of block I+1.  The CTA
// computes r on its 32 x 8 tile and on the high ring the tangential in-plane
// axes need into shared memory (Rs), evaluates the ring positions that lie
// on a domain ghost as the homogenized BC image of r (faces, then the
// corner from the face ghost: fill_ghosts' last-axis-first chain,
// PKG/boundary.py:90-156) and the P box's ghost corner likewise under the
// true BC (its face pads are kept current by the sweeps); then restricts.
//  * EA = 0: both tangential axes (1 outer, 2 inner) are in-plane: coarse
//    plane b0 comes from fine plane b0 (planes b0 <= B0-1; B0 holds the wall).
//  * EA = 1, 2: the outer tangential axis is the march axis: the inner
//    (in-plane) sums of plane b0 are carried in registers and coarse plane
//    b0-1 completes at step b0 with the first class of plane b0 (the chunk
//    marches one plane further; plane B0+1 is the axis-0 ghost, evaluated
//    from plane B0's values as the BC image).
// Arithmetic: residual as k_resid_tma (op_fast's order), restriction as
// restrict_edge_pt -- bitwise.
namespace esw {
constexpr int TX = 32, TY = 8, HX = TX + 4, HB = 384;
constexpr size_t SLOT = (size_t)8 * HB;
constexpr size_t SMEM = (3 * SLOT) * 8 + 2 * 8;  // 2 box slots + Rs
constexpr unsigned TXB = 8u * HX * (TY + 2) * 8u;
}  // namespace esw

__device__ __forceinline__ double img_bc(const BcSpec& bc, int a, double v) {
    // BC image across the HIGH face of axis a: Dirichlet 2g - v, else v
    int k;
    double g;
    if (a == 0) { k = bc.kind[0][1]; g = bc.val[0][1]; }
    else if (a == 1) { k = bc.kind[1][1]; g = bc.val[1][1]; }
    else { k = bc.kind[2][1]; g = bc.val[2][1]; }
    return k == BC_DIRICHLET ? sb(ml(2.0, g), v) : v;
}

template <int EA>
__global__ void __launch_bounds__(256, 2) k_tau_edge_tma(const __grid_constant__ CUtensorMap mapH,
                                                      double* __restrict__ P,
                                                      const double* __restrict__ F, Lvl L,
                                                      BcSpec bc, BcSpec bch, int chunk,
                                                      double* __restrict__ Pc,
                                                      double* __restrict__ Fc, Lvl Lc,
                                                      double* __restrict__ PIc) {
    using namespace esw;
    static_assert(EA >= 0 && EA <= 2, "edge axis");
    // tangential axes: outer TO, inner TI (restrict_edge_pt's P1, P2)
    constexpr int TO = EA == 0 ? 1 : 0, TI = EA == 2 ? 1 : 2;
    constexpr int BE = 4 >> EA, BO = 4 >> TO, BI = 4 >> TI;  // class bits
    constexpr bool CARRY = EA != 0;  // outer axis = march axis
    extern __shared__ __align__(128) double sm[];
    double* Rs = sm + 2 * SLOT;
    unsigned long long* bar = (unsigned long long*)(sm + 3 * SLOT);
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
    const int x0 = blockIdx.x * TX + 1, y0 = blockIdx.y * TY + 1;
    const int b0s = 1 + blockIdx.z * chunk;
    const int b0e = min(L.B[0], b0s + chunk - 1);
    const int B0 = L.B[0], B1 = L.B[1], B2 = L.B[2];
    const int last = CARRY ? b0e + 1 : b0e;  // last march step
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
    const bool active = b1 <= B1 && b2 <= B2;
    const int ci = (ty + 1) * HX + tx + 2;  // tile centre in a box
    // residual of class c at box position q (block (b0, y0-1+q/HX, x0-2+q%HX));
    // v0 = its across-face axis-0 neighbour (direct global load)
    auto resid = [&](const double* S, int c, int q, double fv, double v0) {
        const double pc = S[c * HB + q];
        double ns = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int bit = 1 << (2 - a);
            const bool qa = (c & bit) != 0;
            const int k = c ^ bit;
            const double inside = S[k * HB + q];
            const double out = a == 0 ? v0 : S[k * HB + q + (a == 1 ? (qa ? -HX : HX) : (qa ? -1 : 1))];
            const double e = qa ? inside : out, w = qa ? out : inside;
            ns = a == 0 ? ad(e, w) : ad(ad(ns, e), w);
        }
        const double lap = ml(sb(ns, ml(6.0, pc)), L.inv_h2);
        return sb(fv, sb(ml(L.a, pc), ml(L.b, lap)));
    };
    // (CARRY) inner sums of the previous plane: [cI][outer bit 1 / 0], p and r
    double zp[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, zr[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    // f and the across-face axis-0 neighbour of every class of the tile
    // block, loaded straight from global one step AHEAD (in flight while
    // the previous plane is restricted); the extra step needs classes 4..7
    double fv[8], nb0[8];
    auto load_tile = [&](int b0) {
        const unsigned need = (CARRY && b0 == b0e + 1) ? 0xF0u : 0xFFu;
        const long o = at<3>(L, 0, b0, b1, b2);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            fv[c] = 0.0;
            nb0[c] = 0.0;
            if (!active || !((need >> c) & 1u)) continue;
            fv[c] = __ldg(F + o + (long)c * L.cls);
            const int k = c ^ 4;
            nb0[c] = P[o + (long)k * L.cls + ((k & 4) ? L.s0 : -L.s0)];
        }
    };
    // high ring along the in-plane tangential axes: (position, class) items
    // of the classes with the ring axis' bit set, one per thread; their f
    // and axis-0 neighbour are loaded one step ahead too
    constexpr int NROW = TO == 1 || TI == 1 ? TX : 0;  // ring row (axis 1)
    constexpr int NCOL = TO == 2 || TI == 2 ? TY : 0;  // ring column (axis 2)
    constexpr int NCOR = (NROW && NCOL) ? 1 : 0;
    constexpr int NITEM = 4 * NROW + 4 * NCOL + 2 * NCOR;
    int iq = -1, ic = 0;
    double ifv = 0.0, inb = 0.0;
    auto load_ring = [&](int b0) {
        iq = -1;
        if (tid >= NITEM) return;
        const bool ext = CARRY && b0 == b0e + 1;
        int rb1, rb2, j = tid & 3, cand;
        if (tid < 4 * NROW) { rb1 = y0 + TY; rb2 = x0 + (tid >> 2); cand = 2; }
        else if (tid < 4 * NROW + 4 * NCOL) { const int t = tid - 4 * NROW; rb1 = y0 + (t >> 2); rb2 = x0 + TX; cand = 1; }
        else { rb1 = y0 + TY; rb2 = x0 + TX; cand = 3; j = tid - 4 * NROW - 4 * NCOL; }
        // the j-th class with all `cand` bits set (and outer bit 1 on the extra step)
        int n = 0;
#pragma unroll
        for (int c = 0; c < 8; ++c)
            if ((c & cand) == cand && (!ext || (c & 4))) {
                if (n == j) ic = c;
                ++n;
            }
        if (j < n && rb1 <= B1 && rb2 <= B2) {  // interior ring position
            iq = (rb1 - (y0 - 1)) * HX + (rb2 - (x0 - 2));
            const long o = at<3>(L, 0, b0, rb1, rb2);
            ifv = __ldg(F + o + (long)ic * L.cls);
            const int k = ic ^ 4;
            inb = P[o + (long)k * L.cls + ((k & 4) ? L.s0 : -L.s0)];
        }
    };
    load_tile(b0s);
    load_ring(b0s);
    for (int b0 = b0s; b0 <= last; ++b0) {
        const int s = (b0 - b0s) & 1;
        const bool ghost = CARRY && b0 == B0 + 1;       // axis-0 ghost plane
        const bool extra = CARRY && b0 == b0e + 1;      // only outer-bit-1 classes needed
        if (tid == 0 && b0 < last && !(CARRY && b0 + 1 == B0 + 1)) issue(b0 + 1, s ^ 1);
        const double* S = sm + (ghost ? (s ^ 1) : s) * SLOT;  // ghost step: plane B0's box
        double own_p[8], own_r[8];  // the tile block's p and r (regular steps)
        if (!ghost) {
            const unsigned cls_need = extra ? 0xF0u : 0xFFu;  // bit 0 set: classes 4..7
            mbar_wait(&bar[s], ((b0 - b0s) >> 1) & 1);
            if (active) {
                // the block's 8 p values once (k_resid_tma's pattern): the
                // inside neighbours come from registers, only the across-face
                // in-plane ones from the box
#pragma unroll
                for (int c = 0; c < 8; ++c) own_p[c] = S[c * HB + ci];
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    own_r[c] = 0.0;
                    if (!((cls_need >> c) & 1u)) continue;
                    int bb[3] = {b0, b1, b2};
                    if (is_wall<3, EA>(L, c, bb)) continue;  // not an unknown (never restricted)
                    double ns = 0.0;
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        const int bit = 1 << (2 - a);
                        const bool qa = (c & bit) != 0;
                        const int k = c ^ bit;
                        const double out = a == 0 ? nb0[c]
                                                  : S[k * HB + ci + (a == 1 ? (qa ? -HX : HX) : (qa ? -1 : 1))];
                        const double e = qa ? own_p[k] : out, w = qa ? out : own_p[k];
                        ns = a == 0 ? ad(e, w) : ad(ad(ns, e), w);
                    }
                    const double lap = ml(sb(ns, ml(6.0, own_p[c])), L.inv_h2);
                    own_r[c] = sb(fv[c], sb(ml(L.a, own_p[c]), ml(L.b, lap)));
                    Rs[c * HB + ci] = own_r[c];
                }
            }
            if (iq >= 0) Rs[ic * HB + iq] = resid(S, ic, iq, ifv, inb);
            if (b0 < last && !(CARRY && b0 + 1 == B0 + 1)) {
                load_tile(b0 + 1);
                load_ring(b0 + 1);
            }
            __syncthreads();
            // ghosts of the ring on the high domain faces, last axis first
            // (faces of axis 2, then axis 1 incl. the corner): r under the
            // homogenized bc; the P box only needs its corner (face pads are
            // current in memory).  Only tiles touching a high face.
            const bool gcol = NCOL && x0 + TX - 1 >= B2, grow = NROW && y0 + TY - 1 >= B1;
            if (gcol && tid < TY + 1) {  // column B2+1
                const int r = tid + 1, q = B2 + 1 - (x0 - 2);
                if (y0 - 1 + r <= B1 + 1)
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        if (c & 1) Rs[c * HB + r * HX + q] = img_bc(bch, 2, Rs[(c ^ 1) * HB + r * HX + q - 1]);
            }
            if (gcol && grow) __syncthreads();  // the corner reads the column
            if (grow && tid < TX + 1) {  // row B1+1
                const int r = B1 + 1 - (y0 - 1), q = tid + 2;
                if (x0 - 2 + q <= B2 + 1)
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        if (c & 2) {
                            Rs[c * HB + r * HX + q] = img_bc(bch, 1, Rs[(c ^ 2) * HB + (r - 1) * HX + q]);
                            if (NCOL && x0 - 2 + q == B2 + 1 && (c & 1))  // P box corner
                                ((double*)S)[c * HB + r * HX + q] =
                                    img_bc(bc, 1, S[(c ^ 2) * HB + (r - 1) * HX + q]);
                        }
            }
            if (gcol || grow) __syncthreads();
        }
        // ---- restriction ----
        // own-block values from registers, the +1 blocks along the
        // tangential axes from Rs / the box; on the axis-0 ghost plane (CARRY,
        // last chunk) every value is the BC image of plane B0's class c^4
        auto rv = [&](int c, int q) {
            return ghost ? img_bc(bch, 0, Rs[(c ^ 4) * HB + q]) : Rs[c * HB + q];
        };
        auto pv = [&](int c, int q) {
            return ghost ? img_bc(bc, 0, S[(c ^ 4) * HB + q]) : S[c * HB + q];
        };
        // inner (1,2,1)/4 over TI: classes e|BI, e of this block and e|BI of
        // the next block along TI (restrict_edge_pt's F(.., dk))
        constexpr int DQ = TI == 2 ? 1 : HX;
        auto zown = [&](const double* own, const double* A, int e) {
            return ml(ad(ad(own[e | BI], ml(2.0, own[e])), A[(e | BI) * HB + ci + DQ]), 0.25);
        };
        if (!CARRY) {
            // coarse plane b0 (edge axis 0: planes 1..B0-1); TO = 1, TI = 2
            if (active && b0 <= B0 - 1) {
                double res[2];
#pragma unroll
                for (int w = 0; w < 2; ++w) {
                    const double* own = w ? own_p : own_r;
                    const double* A = w ? S : Rs;
                    double tang[2];
#pragma unroll
                    for (int cI = 0; cI < 2; ++cI) {
                        const int e = cI == 0 ? BE : 0;
                        const double r0 = zown(own, A, e | BO);
                        const double r1 = zown(own, A, e);
                        // row 2J+1: class e|BO of the next block along axis 1
                        const int q2 = ci + HX;
                        const double r2 = ml(ad(ad(A[(e | BO | BI) * HB + q2], ml(2.0, A[(e | BO) * HB + q2])),
                                                A[(e | BO | BI) * HB + q2 + 1]), 0.25);
                        tang[cI] = ml(ad(ad(r0, ml(2.0, r1)), r2), 0.25);
                    }
                    res[w] = ml(ad(tang[0], tang[1]), 0.5);
                }
                int bb[3] = {b0, b1, b2}, cc = 0, cb3[3] = {0, 0, 0};
                coarse_of<3>(L, Lc, bb, cc, cb3);
                const long oc = at<3>(Lc, cc, cb3[0], cb3[1], cb3[2]);
                Pc[oc] = res[1];
                PIc[oc] = res[1];
                Fc[oc] = res[0];
            }
        } else {
            // inner sums of this plane (outer bit 1; bit 0 too except on the
            // extra/ghost step), then coarse plane b0-1 from the carry
            const bool edge_ok = active && (EA == 1 ? b1 <= B1 - 1 : b2 <= B2 - 1);
            if (edge_ok) {
                double tr[2], tp[2];
#pragma unroll
                for (int cI = 0; cI < 2; ++cI) {
                    const int e = cI == 0 ? BE : 0;
                    // row 2J+1 of coarse plane b0-1 = this plane's first
                    // class; then this plane's sums become the carry
                    double r1, p1;
                    if (ghost) {
                        const int c0 = e | BO;
                        r1 = ml(ad(ad(rv(c0 | BI, ci), ml(2.0, rv(c0, ci))), rv(c0 | BI, ci + DQ)), 0.25);
                        p1 = ml(ad(ad(pv(c0 | BI, ci), ml(2.0, pv(c0, ci))), pv(c0 | BI, ci + DQ)), 0.25);
                    } else {
                        r1 = zown(own_r, Rs, e | BO);
                        p1 = zown(own_p, S, e | BO);
                    }
                    tr[cI] = ml(ad(ad(zr[cI][0], ml(2.0, zr[cI][1])), r1), 0.25);
                    tp[cI] = ml(ad(ad(zp[cI][0], ml(2.0, zp[cI][1])), p1), 0.25);
                    zr[cI][0] = r1;
                    zp[cI][0] = p1;
                    if (!extra && !ghost) {
                        zr[cI][1] = zown(own_r, Rs, e);
                        zp[cI][1] = zown(own_p, S, e);
                    }
                }
                if (b0 > b0s) {
                    int bb[3] = {b0 - 1, b1, b2}, cc = 0, cb3[3] = {0, 0, 0};
                    coarse_of<3>(L, Lc, bb, cc, cb3);
                    const long oc = at<3>(Lc, cc, cb3[0], cb3[1], cb3[2]);
                    const double pres = ml(ad(tp[0], tp[1]), 0.5);
                    Pc[oc] = pres;
                    PIc[oc] = pres;
                    Fc[oc] = ml(ad(tr[0], tr[1]), 0.5);
                }
            }
        }
        __syncthreads();  // box slot s and Rs are refilled next step
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
                if ((MASK >> c) & 1u) nv[c] = dvr(nv[c], L.denom, L.rden);
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
