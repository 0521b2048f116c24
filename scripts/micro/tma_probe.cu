// Minimal TMA 4D tile-load probe (debugging the wave kernel's loads).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap m, double* out, int x, int y, int z, int c, int mode, const double* src) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        if (mode & 4) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(34 * 9 * 8) : "memory");
        if (mode & 8)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su32(sm)), "l"(src), "r"(34 * 9 * 8), "r"(su32(&bar)) : "memory");
        else if ((mode & 1) == 0)
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                         ::"r"(su32(sm)), "l"((unsigned long long)&m), "r"(x), "r"(y), "r"(z), "r"(c), "r"(su32(&bar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                         ::"r"(su32(sm)), "l"((unsigned long long)&m), "r"(x), "r"(y), "r"(z), "r"(c), "r"(su32(&bar)) : "memory");
    }
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}" ::"r"(su32(&bar)) : "memory");
    for (int i = threadIdx.x; i < 34 * 9; i += blockDim.x) out[i] = sm[i];
}
#include <cstdlib>
int main(int argc, char** argv) {
    const long pitch = 40, E1 = 12, E0 = 12, cls = pitch * E1 * E0;
    std::vector<double> h(cls * 8);
    for (long i = 0; i < (long)h.size(); ++i) h[i] = (double)i;
    double *d, *o;
    cudaMalloc(&d, h.size() * 8); cudaMalloc(&o, 34 * 9 * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    CUtensorMap m;
    cuuint64_t dims[4] = {(cuuint64_t)pitch, (cuuint64_t)E1, (cuuint64_t)E0, 8};
    cuuint64_t st[3] = {(cuuint64_t)pitch * 8, (cuuint64_t)pitch * E1 * 8, (cuuint64_t)cls * 8};
    cuuint32_t box[4] = {34, 9, 1, 1}, es[4] = {1, 1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d q %d\n", (int)r, (int)q);
    int dt = argc > 2 ? atoi(argv[2]) : 0;
    if (dt) {
        r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_INT64, 4, d, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("encode int64 %d\n", (int)r);
    }
    for (int mode = atoi(argv[1]); mode <= atoi(argv[1]); ++mode) {
        k<<<1, 128, 4096>>>(m, o, 3, 1, 2, 5, mode, d);
        cudaError_t e = cudaDeviceSynchronize();
        printf("mode %d: %s\n", mode, cudaGetErrorString(e));
        if (e) return 1;
        std::vector<double> out(34 * 9);
        cudaMemcpy(out.data(), o, out.size() * 8, cudaMemcpyDeviceToHost);
        long base = 5 * cls + 2 * pitch * E1 + 1 * pitch + 3;
        int bad = 0;
        for (int yy = 0; yy < 9; ++yy) for (int xx = 0; xx < 34; ++xx) {
            long gi = base + yy * pitch + xx;
            double want = (3 + xx < pitch && 1 + yy < E1) ? (double)gi : 0.0;
            if (out[yy * 34 + xx] != want) ++bad;
        }
        printf("mode %d mismatches %d\n", mode, bad);
    }
    return 0;
}
