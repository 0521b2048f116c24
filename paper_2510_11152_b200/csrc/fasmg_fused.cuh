// fasmg_fused.cuh -- the last smoothing half-sweep of a level fused with the
// residual that follows it (included by fasmg_engine.cu inside namespace
// fasmg, after fasmg_wave.cuh).
//
// In the FAS V-cycle the residual r = f - L(p) is evaluated right after the
// last smoothing half-sweep of a level twice: by the tau pass (descent,
// PKG/fas.py:98-110) and by the outer residual norm after the V-cycle
// (PKG/fas.py:149-151).  Separately those are a 12 B/DOF half-sweep plus a
// 16 B/DOF residual pass.  Fused, the only extra HBM traffic is f of the
// other color (4 B/DOF): the residual of plane b0-1 is formed while its
// neighbourhood is still in shared memory.
//
// A CTA owns a 32 (b2) x 8 (b1) tile and marches a chunk of planes.  At step
// j it
//   1. runs the half-sweep (color B = MASK) at plane j on the tile AND its
//      1-block in-plane ring -- the ring values belong to neighbouring tiles
//      and are recomputed here from identical inputs, so they are bitwise
//      what their owners store -- needing color A (the opposite classes)
//      with a 2-block ring; A boxes are 36 x 12 TMA loads;
//   2. stores the tile's new B values to global memory and mirrors the
//      ghost updates of boundary B points into the shared A planes (a
//      ghost of a B point lives in an A-class pad slot).  The global ghost
//      pads are refreshed by k_pad_fill after the kernel: a ring point's
//      pre-sweep ghost must stay readable by every CTA until all are done;
//   3. evaluates the residual of all 2^3 classes at plane j-1 of the tile
//      (A and new B at planes j-2..j, f of both colors at j-1) and either
//      accumulates sum(r^2) (MODE_NORM) or restricts r and p to the coarse
//      cell of each block and writes p_c, f_c with coarse pads (MODE_TAU,
//      the arithmetic of tau_pt).
// Boundary tiles also load the B classes' own pad slots (ghosts of A
// points, untouched by this kernel) into a separate staging ring.  Per-point arithmetic is exactly sweep_pt's /
// tau_pt's, so fields are bitwise equal; only the norm's summation order
// changes (a different fixed tree, ~1e-16 relative).  Cell-centred fields
// with Dirichlet/Neumann faces (periodic wraps would couple distant tiles).
#pragma once

namespace fsw {
constexpr int TX = 32, TY = 8;
constexpr int AX = TX + 4, AY = TY + 4;   // A / B plane box: cols x0-2..x0+33, rows y0-2..y0+9
constexpr int AB = 448;                   // doubles per box slot (432 -> 128 B multiple)
constexpr int FX = TX + 4, FY = TY + 2;   // f of B: cols x0-2..x0+33, rows y0-1..y0+8
constexpr int FB = 384;                   // (360 -> 128 B multiple)
constexpr int FA = TX * TY;               // f of A: the tile
constexpr int RA = 5, RF = 3, RFA = 2, RB = 3;
constexpr size_t OFF_A = 0;
constexpr size_t OFF_B = OFF_A + (size_t)4 * RA * AB;
constexpr size_t OFF_FB = OFF_B + (size_t)4 * RB * AB;
constexpr size_t OFF_FA = OFF_FB + (size_t)4 * RF * FB;
constexpr size_t OFF_PAD = OFF_FA + (size_t)4 * RFA * FA;   // B classes' pad slots
constexpr size_t OFF_RED = OFF_PAD + (size_t)4 * RB * AB;
constexpr size_t SMEM = (OFF_RED + 256) * 8 + 4 * 8;
constexpr unsigned ABYTES = AX * AY * 8u, FBYTES = FX * FY * 8u, FABYTES = FA * 8u;
enum { MODE_NORM = 0, MODE_TAU = 1 };
}  // namespace fsw

template <int MODE, unsigned MASK>
__global__ void __launch_bounds__(256, 1)
    k_sweep_resid(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapFB,
                  const __grid_constant__ CUtensorMap mapFA, double* __restrict__ P, Lvl L,
                  BcSpec bc, int chunk, double* __restrict__ part, double* __restrict__ Pc,
                  double* __restrict__ Fc, Lvl Lc) {
    using namespace fsw;
    constexpr unsigned OPP = MASK ^ 0xFFu;
    extern __shared__ __align__(128) double sm[];
    double* sA = sm + OFF_A;     // [4 A classes][RA planes][AB]
    double* sB = sm + OFF_B;     // [4 B classes][RB planes][AB]
    double* sFB = sm + OFF_FB;   // [4][RF][FB]
    double* sFA = sm + OFF_FA;   // [4][RFA][FA]
    double* sPad = sm + OFF_PAD; // [4 B classes][RB planes][AB]: B boxes, read at pad slots only
    double* red = sm + OFF_RED;
    unsigned long long* bar = (unsigned long long*)(red + 256);  // [0,1] prefetch, [2] B pads
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
    const int x0 = blockIdx.x * TX + 1, y0 = blockIdx.y * TY + 1;
    const int B0 = L.B[0], B1 = L.B[1], B2 = L.B[2];
    const int b0s = 1 + blockIdx.z * chunk;
    const int b0e = min(B0, b0s + chunk - 1);
    // tiles whose ring touches an in-plane pad need the B classes' pad slots
    const bool edge_tile = y0 == 1 || x0 == 1 || y0 + TY > B1 || x0 + TX > B2;

    auto slotA = [&](int k, int pl) { return sA + (oslot<OPP>(k) * RA + (pl + RA) % RA) * AB; };
    auto slotB = [&](int k, int pl) { return sB + (oslot<MASK ^ 0u>(k) * RB + (pl + RB) % RB) * AB; };
    auto slotP = [&](int k, int pl) { return sPad + (oslot<MASK ^ 0u>(k) * RB + (pl + RB) % RB) * AB; };
    auto issue_A = [&](int pl, unsigned long long* br) {
        for (int k = 0; k < 8; ++k)
            if ((OPP >> k) & 1u)
                tma_load4(slotA(k, pl), &mapA, br, OFF + x0 - 2, y0 - 2, pl, k);
    };
    auto issue_FB = [&](int pl, unsigned long long* br) {
        int j = 0;
        for (int k = 0; k < 8; ++k)
            if ((MASK >> k) & 1u) {
                tma_load4(sFB + (j * RF + pl % RF) * FB, &mapFB, br, OFF + x0 - 2, y0 - 1, pl, k);
                ++j;
            }
    };
    auto issue_FA = [&](int pl, unsigned long long* br) {
        int j = 0;
        for (int k = 0; k < 8; ++k)
            if ((OPP >> k) & 1u) {
                tma_load4(sFA + (j * RFA + pl % RFA) * FA, &mapFA, br, OFF + x0, y0, pl, k);
                ++j;
            }
    };

    const int jfirst = b0s - 1, jlast = b0e + 1;
    if (tid == 0) {
        for (int i = 0; i < 3; ++i) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // prologue (for step jfirst): A planes jfirst-1..jfirst+1, f_B plane jfirst
        unsigned long long* br = &bar[jfirst & 1];
        unsigned bytes = 0;
        for (int pl = jfirst - 1; pl <= jfirst + 1; ++pl)
            if (pl >= 0 && pl <= B0 + 1) bytes += 4 * ABYTES;
        if (jfirst >= 1) bytes += 4 * FBYTES;
        mbar_expect_tx(br, bytes);
        for (int pl = jfirst - 1; pl <= jfirst + 1; ++pl)
            if (pl >= 0 && pl <= B0 + 1) issue_A(pl, br);
        if (jfirst >= 1) issue_FB(jfirst, br);
    }
    __syncthreads();

    double acc = 0.0;
    unsigned phB = 0;
    for (int j = jfirst; j <= jlast; ++j) {
        const bool pad_plane = j < 1 || j > B0;
        if (tid == 0) {
            // slots about to be refilled by TMA were last written by generic
            // stores (new B values, mirrored ghosts): order the proxies
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            // prefetch for step j+1: A plane j+2, f_B plane j+1, f_A plane j
            if (j < jlast) {
                unsigned long long* br = &bar[(j + 1) & 1];
                unsigned bytes = 0;
                const bool a2 = j + 2 <= B0 + 1, fb1 = j + 1 >= 1 && j + 1 <= B0,
                           fa0 = j >= b0s && j <= b0e;
                bytes = (a2 ? 4 * ABYTES : 0) + (fb1 ? 4 * FBYTES : 0) + (fa0 ? 4 * FABYTES : 0);
                mbar_expect_tx(br, bytes);
                if (a2) issue_A(j + 2, br);
                if (fb1) issue_FB(j + 1, br);
                if (fa0) issue_FA(j, br);  // (bytes == 0: the arrive completes the phase)
            }
            // the B classes' own pad slots of plane j (pad plane: all of it)
            if (pad_plane || edge_tile) {
                mbar_expect_tx(&bar[2], 4 * ABYTES);
                for (int k = 0; k < 8; ++k)
                    if ((MASK >> k) & 1u)
                        tma_load4(slotP(k, j), &mapA, &bar[2], OFF + x0 - 2, y0 - 2, j, k);
            }
        }
        mbar_wait(&bar[j & 1], ((j - jfirst) >> 1) & 1);
        if (pad_plane || edge_tile) {
            mbar_wait(&bar[2], phB);
            phB ^= 1u;
        }
        // ---- 1+2. half-sweep of color B at plane j on tile + 1-ring
        if (!pad_plane) {
            for (int e = tid; e < (TY + 2) * (TX + 2); e += TX * TY) {
                const int r = e / (TX + 2), q = e - r * (TX + 2);
                const int b1 = y0 - 1 + r, b2 = x0 - 1 + q;
                if (b1 < 1 || b1 > B1 || b2 < 1 || b2 > B2) continue;
                const int ci = (r + 1) * AX + (q + 1);  // (b1, b2) in a 36 x 12 box
                const int fi = r * FX + (q + 1);        // (b1, b2) in the f_B box
                double nv[8];
                int jj = 0;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    if (!((MASK >> c) & 1u)) continue;
                    const int k0 = c ^ 4, k1 = c ^ 2, k2 = c ^ 1;
                    const int lo0 = (k0 & 4) ? j : j - 1;
                    const double e0 = slotA(k0, lo0 + 1)[ci], w0 = slotA(k0, lo0)[ci];
                    const double* w1p = slotA(k1, j);
                    const double* w2p = slotA(k2, j);
                    const bool q1 = (c & 2) != 0, q2 = (c & 1) != 0;
                    const double e1 = w1p[ci + (q1 ? 0 : AX)], w1 = w1p[ci - (q1 ? AX : 0)];
                    const double e2 = w2p[ci + (q2 ? 0 : 1)], w2 = w2p[ci - (q2 ? 1 : 0)];
                    double ns = ad(e0, w0);
                    ns = ad(ad(ns, e1), w1);
                    ns = ad(ad(ns, e2), w2);
                    nv[c] = ad(ml(L.h2, sFB[(jj * RF + j % RF) * FB + fi]), ml(L.b, ns));
                    ++jj;
                }
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    if ((MASK >> c) & 1u) nv[c] = dv(nv[c], L.denom);
                int bb[3] = {j, b1, b2};
                const bool own = r >= 1 && r <= TY && q >= 1 && q <= TX && j >= b0s && j <= b0e;
                const bool bnd = on_boundary<3>(L, bb);
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    if (!((MASK >> c) & 1u)) continue;
                    slotB(c, j)[ci] = nv[c];
                    // global ghost pads are NOT refreshed here: other CTAs
                    // may still load the pre-sweep ghosts of ring points;
                    // the host runs k_pad_fill right after this kernel
                    if (own) P[at<3>(L, c, j, b1, b2)] = nv[c];
                    if (bnd) {
                        // mirror write_pads into the shared A planes
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            const int bit = 1 << (2 - a);
                            const bool qa = (c & bit) != 0;
                            const int g = bb[a], Bn = a == 0 ? B0 : (a == 1 ? B1 : B2);
                            const int side = (qa && g == 1) ? 0 : ((!qa && g == Bn) ? 1 : -1);
                            if (side < 0) continue;
                            const int kk = bc.kind[a][side];
                            const double gv = kk == BC_DIRICHLET ? sb(ml(2.0, bc.val[a][side]), nv[c])
                                                                 : nv[c];
                            const int d = side == 0 ? -1 : 1;
                            if (a == 0) slotA(c ^ bit, j + d)[ci] = gv;
                            else if (a == 1) slotA(c ^ bit, j)[ci + d * AX] = gv;
                            else slotA(c ^ bit, j)[ci + d] = gv;
                        }
                    }
                }
            }
        }
        __syncthreads();
        // ---- 3. residual of all classes at plane j-1 on the tile
        const int pr = j - 1;
        if (pr >= b0s && pr <= b0e) {
            const int b1 = y0 + ty, b2 = x0 + tx;
            if (b1 <= B1 && b2 <= B2) {
                const int ci = (ty + 2) * AX + (tx + 2);
                // value of class k at plane pl, in-plane offset (d1, d2)
                auto val = [&](int k, int pl, int d1, int d2) {
                    if ((OPP >> k) & 1u) return slotA(k, pl)[ci + d1 * AX + d2];
                    const int g1 = b1 + d1, g2 = b2 + d2;
                    const bool pad = pl < 1 || pl > B0 || g1 < 1 || g1 > B1 || g2 < 1 || g2 > B2;
                    return (pad ? slotP(k, pl) : slotB(k, pl))[ci + d1 * AX + d2];
                };
                double pc[8], fv[8];
                int ja = 0, jb = 0;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    pc[c] = val(c, pr, 0, 0);
                    if ((OPP >> c) & 1u) {
                        fv[c] = sFA[(ja * RFA + pr % RFA) * FA + tid];
                        ++ja;
                    } else {
                        fv[c] = sFB[(jb * RF + pr % RF) * FB + (ty + 1) * FX + (tx + 2)];
                        ++jb;
                    }
                }
                double rp = 0.0, rr = 0.0;
#pragma unroll
                for (int c = 7; c >= 0; --c) {
                    double ns = 0.0;
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        const int bit = 1 << (2 - a);
                        const bool qa = (c & bit) != 0;
                        // neighbour class c^bit: same block (inside) or the
                        // adjacent block across the face (W of q=1, E of q=0)
                        const double inside = pc[c ^ bit];
                        const int s = qa ? -1 : 1;
                        const double out = a == 0 ? val(c ^ bit, pr + s, 0, 0)
                                                  : (a == 1 ? val(c ^ bit, pr, s, 0)
                                                            : val(c ^ bit, pr, 0, s));
                        const double e = qa ? inside : out;
                        const double w = qa ? out : inside;
                        ns = a == 0 ? ad(e, w) : ad(ad(ns, e), w);
                    }
                    const double lap = ml(sb(ns, ml(6.0, pc[c])), L.inv_h2);
                    const double r = sb(fv[c], sb(ml(L.a, pc[c]), ml(L.b, lap)));
                    if (MODE == MODE_NORM) {
                        acc = ad(acc, ml(r, r));
                        if (Fc) Fc[at<3>(L, c, pr, b1, b2)] = r;  // debug: per-point residual
                    } else {
                        if (c == 7) { rp = pc[c]; rr = r; }
                        else { rp = ad(rp, pc[c]); rr = ad(rr, r); }
                    }
                }
                if (MODE == MODE_TAU) {
                    int bb[3] = {pr, b1, b2}, cc = 0, cb[3] = {0, 0, 0};
                    coarse_of<3>(L, Lc, bb, cc, cb);
                    const long oc = at<3>(Lc, cc, cb[0], cb[1], cb[2]);
                    const double pcv = ml(rp, 0.125);
                    Pc[oc] = pcv;
                    Fc[oc] = ml(rr, 0.125);
                    if (on_boundary<3>(Lc, cb)) write_pads<3, -1>(Pc, Lc, bc, cc, cb, oc, pcv);
                }
            }
        }
        // generic-proxy smem writes of this step (new B values, mirrored
        // ghosts) must be ordered before later TMA refills of those slots:
        // every writing thread fences, then the CTA barrier
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();  // next step's prefetch overwrites this step's oldest slots
    }
    if (MODE == MODE_NORM) {  // fixed-order tree over the CTA
        red[tid] = acc;
        __syncthreads();
        for (int s = 128; s > 0; s >>= 1) {
            if (tid < s) red[tid] = ad(red[tid], red[tid + s]);
            __syncthreads();
        }
        if (tid == 0) part[blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)] = red[0];
    }
}
