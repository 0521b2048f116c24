// fasmg_runtime.cu -- error state, stream helpers and library metadata for
// the C ABI (include/fasmg_b200.h).
#include <stdio.h>
#include <string.h>

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

}  // extern "C"
