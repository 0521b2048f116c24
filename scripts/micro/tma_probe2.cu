// TMA variants probe: param-space vs global-memory descriptor, 2D vs 4D, box shapes.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap m, const CUtensorMap* gm, double* out, int rank, int useg, unsigned bytes, int c0, int c1, int c2, int c3) {
    extern __shared__ __align__(1024) double sm[];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long mp = useg ? (unsigned long long)gm : (unsigned long long)&m;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes) : "memory");
        if (rank == 4)
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                         ::"r"(su32(sm)), "l"(mp), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(su32(&bar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(su32(sm)), "l"(mp), "r"(0), "r"(0), "r"(su32(&bar)) : "memory");
    }
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}" ::"r"(su32(&bar)) : "memory");
    if (threadIdx.x == 0) out[0] = sm[1];
}
int main(int argc, char** argv) {
    int rank = atoi(argv[1]), useg = atoi(argv[2]), bx = atoi(argv[3]), by = atoi(argv[4]), dt = atoi(argv[5]);
    const long pitch = 64, E1 = 16, E0 = 16, cls = pitch * E1 * E0;
    double *d, *o; CUtensorMap* gm;
    cudaMalloc(&d, cls * 8 * 8); cudaMalloc(&o, 8); cudaMalloc(&gm, sizeof(CUtensorMap));
    cudaMemset(d, 0, cls * 64);
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    CUtensorMap m;
    cuuint64_t dims[4] = {(cuuint64_t)pitch, (cuuint64_t)E1, (cuuint64_t)E0, 8};
    cuuint64_t st[3] = {(cuuint64_t)pitch * 8, (cuuint64_t)pitch * E1 * 8, (cuuint64_t)cls * 8};
    cuuint32_t box[4] = {(cuuint32_t)bx, (cuuint32_t)by, 1, 1}, es[4] = {1, 1, 1, 1};
    CUtensorMapDataType t = dt == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : (dt == 1 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT8);
    int esz = dt == 0 ? 8 : (dt == 1 ? 4 : 1);
    if (dt) { dims[0] = pitch * 8 / esz; }
    CUresult r = enc(&m, t, rank, d, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
    unsigned bytes = bx * by * esz;
    k<<<1, 32, 8192>>>(m, gm, o, rank, useg, bytes, atoi(argv[6]), atoi(argv[7]), atoi(argv[8]), atoi(argv[9]));
    cudaError_t e = cudaDeviceSynchronize();
    printf("c %s %s %s %s rank %d useg %d box %dx%d dt %d: encode %d -> %s\n", argv[6], argv[7], argv[8], argv[9], rank, useg, bx, by, dt, (int)r, cudaGetErrorString(e));
    int drv = 0; cudaDriverGetVersion(&drv); int rt = 0; cudaRuntimeGetVersion(&rt);
    printf("driver %d runtime %d\n", drv, rt);
    return 0;
}
