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
// fields only (edge transfers keep their launches: see coarse_setup).
#pragma once

struct CoarseArgs {
    double* P[32];
    double* F[32];
    Lvl L[32];
    BcSpec bc;
    int k0, k1, nl, s, nm;  // cluster levels k0..k1-1, CTA-0 levels k1..nl-1
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

// Sub-V-cycle over levels ka..nl-1 (descent from ka, coarsest smoothing,
// ascent back to ka), by `gstr` threads with index `gtid`; CL selects the
// barrier between dependent phases: the whole cluster (CL) or this CTA.
template <int D, bool CL>
__device__ __forceinline__ void run_levels(const CoarseArgs* __restrict__ A, int ka, int kb,
                                           bool coarsest, long gtid, long gstr) {
    const BcSpec bc = A->bc;
    const int nl = A->nl;
    auto sync = [] {
        if (CL) cluster_sync_all();
        else __syncthreads();
    };
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
                sync();
            }
    };
    // descent over ka..kb-1 (PKG/fas.py:98-110)
    for (int k = ka; k < kb; ++k) {
        smooth(k);
        const Lvl L = A->L[k], Lc = A->L[k + 1];
        for (long t = gtid; t < L.nblk; t += gstr) {
            int bb[3];
            decode<D>(L, t, bb);
            tau_pt<D>(A->P[k], A->F[k], L, A->P[k + 1], A->F[k + 1], Lc, bc, bb);
        }
        sync();
        for (long t = gtid; t < Lc.nblk; t += gstr) {
            int bb[3];
            decode<D>(Lc, t, bb);
            coarse_src_pt<D, -1>(A->P[k + 1], A->F[k + 1], Lc, bb);
        }
        sync();
    }
    if (coarsest) smooth(nl - 1);  // PKG/fas.py:111-113
    (void)nl;
}

template <int D, bool CL>
__device__ __forceinline__ void run_ascent(const CoarseArgs* __restrict__ A, int ka, int kb,
                                           long gtid, long gstr) {
    const BcSpec bc = A->bc;
    auto sync = [] {
        if (CL) cluster_sync_all();
        else __syncthreads();
    };
    // ascent over kb-1..ka (PKG/fas.py:115-124)
    for (int k = kb - 1; k >= ka; --k) {
        const Lvl L = A->L[k], Lc = A->L[k + 1];
        for (long t = gtid; t < L.nblk; t += gstr) {
            int bb[3];
            decode<D>(L, t, bb);
            correct_pt<D>(A->P[k], L, A->P[k + 1], Lc, bc, bb);
        }
        sync();
        for (int it = 0; it < A->s; ++it)
            for (int j = 0; j < A->nm; ++j) {
                const Lvl Lk = A->L[k];
                for (long t = gtid; t < Lk.nblk; t += gstr) {
                    int bb[3];
                    decode<D>(Lk, t, bb);
                    sweep_dispatch<D>(A->masks[j], A->P[k], A->F[k], Lk, bc, bb);
                }
                sync();
            }
    }
}

// Levels k0..k1-1 run on the whole cluster; levels k1..nl-1 (at most
// ~one block per thread) on CTA 0 alone with CTA barriers, which are an
// order of magnitude cheaper than cluster barriers.
template <int D>
__global__ void __launch_bounds__(512) k_coarse_cycle(const CoarseArgs* __restrict__ A) {
    const unsigned rank = cluster_rank();
    const long gtid = (long)rank * blockDim.x + threadIdx.x;
    const long gstr = (long)cluster_size() * blockDim.x;
    const int k0 = A->k0, k1 = A->k1, nl = A->nl;
    run_levels<D, true>(A, k0, k1, false, gtid, gstr);
    if (rank == 0) {
        run_levels<D, false>(A, k1, nl - 1, true, threadIdx.x, blockDim.x);
        run_ascent<D, false>(A, k1, nl - 1, threadIdx.x, blockDim.x);
    }
    if (k1 > k0) {
        cluster_sync_all();
        run_ascent<D, true>(A, k0, k1, gtid, gstr);
    }
}
