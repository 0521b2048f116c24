// fasmg_runtime.cu -- error state, stream helpers and library metadata for
// the C ABI (include/fasmg_b200.h).
#include <stdio.h>
#include <string.h>

#include "fasmg_common.cuh"
#include "fasmg_internal.h"

static thread_local char g_err[512] = "";
static thread_local int g_code = 0;

int fasmg_set_error(int code, const char* msg) {
    g_code = code;
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}

int fasmg_check(cudaError_t e) {
    if (e == cudaSuccess) return 0;
    char buf[400];
    snprintf(buf, sizeof(buf), "CUDA error %d: %s", (int)e, cudaGetErrorString(e));
    return fasmg_set_error(FASMG_ECUDA, buf);
}

int fasmg_check_launch() { return fasmg_check(cudaGetLastError()); }

extern "C" {

const char* fasmg_last_error(void) { return g_err; }
int fasmg_last_error_code(void) { return g_code; }

int fasmg_version(void) { return 100; }  // 0.1.0

// Architecture this library was compiled for (sm_100a -> 100).
int fasmg_compiled_arch(void) { return 100; }

int fasmg_device_count(int* n) { return fasmg_check(cudaGetDeviceCount(n)); }

int fasmg_stream_create(void** s) {
    cudaStream_t st;
    int r = fasmg_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    *s = (void*)st;
    return r;
}

int fasmg_stream_destroy(void* s) { return fasmg_check(cudaStreamDestroy((cudaStream_t)s)); }

int fasmg_stream_synchronize(void* s) {
    return fasmg_check(cudaStreamSynchronize((cudaStream_t)s));
}

// `waiter` waits (on device) for all work enqueued so far on `signaler`.
int fasmg_stream_wait(void* waiter, void* signaler) {
    cudaEvent_t ev;
    int r = fasmg_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    if (r) return r;
    r = fasmg_check(cudaEventRecord(ev, (cudaStream_t)signaler));
    if (!r) r = fasmg_check(cudaStreamWaitEvent((cudaStream_t)waiter, ev, 0));
    cudaEventDestroy(ev);
    return r;
}

// Self-test of the reciprocal division dvr (fasmg_common.cuh) against
// __ddiv_rn: n numerators per divisor, drawn as random 64-bit patterns
// restricted to normal exponents in [2^-emax, 2^emax] (both signs), plus
// the divisor's own neighbourhood; counts the quotients whose bits differ.
__global__ void k_selftest_div(long n, unsigned long long seed, const double* dens, int nd,
                               int emax, unsigned long long* bad) {
    unsigned long long cnt = 0;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
         i += (long)gridDim.x * blockDim.x) {
        unsigned long long z = seed + (unsigned long long)i * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const unsigned long long mant = z & 0x000FFFFFFFFFFFFFull;
        const int ex = (int)((z >> 52) % (unsigned long long)(2 * emax + 1)) - emax;
        const unsigned long long sgn = (z >> 63) << 63;
        const double a = __longlong_as_double((long long)(sgn | ((unsigned long long)(1023 + ex) << 52) | mant));
        for (int j = 0; j < nd; ++j) {
            const double d = dens[2 * j], r = dens[2 * j + 1];
            const double q = fasmg::dvr(a, d, r), w = __ddiv_rn(a, d);
            cnt += __double_as_longlong(q) != __double_as_longlong(w);
        }
    }
    if (cnt) atomicAdd(bad, cnt);
}

// dens: nd divisors; returns in *bad the number of (numerator, divisor)
// pairs where dvr differs from IEEE division (expected 0)
int fasmg_selftest_div(long n, unsigned long long seed, const double* dens, int nd, int emax,
                       unsigned long long* bad) {
    double* dd = nullptr;
    unsigned long long* db = nullptr;
    double* h = new double[2 * nd];
    for (int j = 0; j < nd; ++j) { h[2 * j] = dens[j]; h[2 * j + 1] = 1.0 / dens[j]; }
    int st = fasmg_check(cudaMalloc(&dd, sizeof(double) * 2 * nd));
    if (!st) st = fasmg_check(cudaMalloc(&db, sizeof(unsigned long long)));
    if (!st) st = fasmg_check(cudaMemcpy(dd, h, sizeof(double) * 2 * nd, cudaMemcpyHostToDevice));
    if (!st) st = fasmg_check(cudaMemset(db, 0, sizeof(unsigned long long)));
    if (!st) {
        k_selftest_div<<<148 * 8, 256>>>(n, seed, dd, nd, emax, db);
        st = fasmg_check_launch();
    }
    if (!st) st = fasmg_check(cudaMemcpy(bad, db, sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    cudaFree(dd);
    cudaFree(db);
    delete[] h;
    return st;
}

}  // extern "C"
