// fasmg_coarse.cuh -- the coarse end of the FAS V-cycle as ONE persistent
// launch (included by fasmg_engine.cu inside namespace fasmg, after
// fasmg_stencil.cuh).
//
// Below a few thousand blocks a level's kernels are pure launch latency
// (~2.5 us each inside a CUDA graph, ~20 per level per V-cycle).  From the
// first such level k0 down to the coarsest, one thread-block cluster (CS
// CTAs on CS SMs) runs the whole sub-cycle of PKG/fas.py:96-128 -- the s
// smoothing steps of every color group, the tau pass (residual +
// restrictions), the coarse source L_2h(R p), the coarsest smoothing and
// the corrections on the way up -- with a cluster barrier
// (barrier.cluster.arrive.release / wait.acquire) between dependent phases
// instead of kernel boundaries.  Each phase is the per-block device function
// of the corresponding standalone kernel (sweep_pt, tau_pt, coarse_src_pt,
// correct_pt in fasmg_stencil.cuh), so the arithmetic and the ghost-pad
// maintenance are identical and results bitwise equal.  Cell-centered
// fields only (edge transfers keep their launches).
#pragma once

struct CoarseArgs {
    double* P[32];
    double* F[32];
    Lvl L[32];
    BcSpec bc;
    int k0, nl, s, nm;
    unsigned masks[16];
};

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile(
        "barrier.cluster.arrive.release.aligned;\n"
        "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_size() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}

template <int D>
__device__ __forceinline__ void sweep_dispatch(unsigned m, double* P, const double* F,
                                               const Lvl& L, const BcSpec& bc, const int* bb) {
    if (D == 3) {
        switch (m) {
            case 0x96u: sweep_pt<3, -1, 0x96u>(P, F, L, bc, bb); return;
            case 0x69u: sweep_pt<3, -1, 0x69u>(P, F, L, bc, bb); return;
            case 0x01u: sweep_pt<3, -1, 0x01u>(P, F, L, bc, bb); return;
            case 0x02u: sweep_pt<3, -1, 0x02u>(P, F, L, bc, bb); return;
            case 0x04u: sweep_pt<3, -1, 0x04u>(P, F, L, bc, bb); return;
            case 0x08u: sweep_pt<3, -1, 0x08u>(P, F, L, bc, bb); return;
            case 0x10u: sweep_pt<3, -1, 0x10u>(P, F, L, bc, bb); return;
            case 0x20u: sweep_pt<3, -1, 0x20u>(P, F, L, bc, bb); return;
            case 0x40u: sweep_pt<3, -1, 0x40u>(P, F, L, bc, bb); return;
            case 0x80u: sweep_pt<3, -1, 0x80u>(P, F, L, bc, bb); return;
        }
    } else {
        switch (m) {
            case 0x6u: sweep_pt<2, -1, 0x6u>(P, F, L, bc, bb); return;
            case 0x9u: sweep_pt<2, -1, 0x9u>(P, F, L, bc, bb); return;
            case 0x1u: sweep_pt<2, -1, 0x1u>(P, F, L, bc, bb); return;
            case 0x2u: sweep_pt<2, -1, 0x2u>(P, F, L, bc, bb); return;
            case 0x4u: sweep_pt<2, -1, 0x4u>(P, F, L, bc, bb); return;
            case 0x8u: sweep_pt<2, -1, 0x8u>(P, F, L, bc, bb); return;
        }
    }
}

template <int D>
__global__ void __launch_bounds__(512) k_coarse_cycle(const CoarseArgs* __restrict__ A) {
    const long gtid = (long)cluster_rank() * blockDim.x + threadIdx.x;
    const long gstr = (long)cluster_size() * blockDim.x;
    const BcSpec bc = A->bc;
    const int k0 = A->k0, nl = A->nl;

    auto smooth = [&](int k) {
        const Lvl L = A->L[k];
        double* P = A->P[k];
        const double* F = A->F[k];
        for (int it = 0; it < A->s; ++it)
            for (int j = 0; j < A->nm; ++j) {
                const unsigned m = A->masks[j];
                for (long t = gtid; t < L.nblk; t += gstr) {
                    int bb[3];
                    decode<D>(L, t, bb);
                    sweep_dispatch<D>(m, P, F, L, bc, bb);
                }
                cluster_sync_all();
            }
    };

    for (int k = k0; k < nl - 1; ++k) {  // descent (PKG/fas.py:98-110)
        smooth(k);
        const Lvl L = A->L[k], Lc = A->L[k + 1];
        for (long t = gtid; t < L.nblk; t += gstr) {
            int bb[3];
            decode<D>(L, t, bb);
            tau_pt<D>(A->P[k], A->F[k], L, A->P[k + 1], A->F[k + 1], Lc, bc, bb);
        }
        cluster_sync_all();
        for (long t = gtid; t < Lc.nblk; t += gstr) {
            int bb[3];
            decode<D>(Lc, t, bb);
            coarse_src_pt<D, -1>(A->P[k + 1], A->F[k + 1], Lc, bb);
        }
        cluster_sync_all();
    }
    smooth(nl - 1);  // coarsest (PKG/fas.py:111-113)
    for (int k = nl - 2; k >= k0; --k) {  // ascent (PKG/fas.py:115-124)
        const Lvl L = A->L[k], Lc = A->L[k + 1];
        for (long t = gtid; t < L.nblk; t += gstr) {
            int bb[3];
            decode<D>(L, t, bb);
            correct_pt<D>(A->P[k], L, A->P[k + 1], Lc, bc, bb);
        }
        cluster_sync_all();
        smooth(k);
    }
}
