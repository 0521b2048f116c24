#include <cuda_runtime.h>
#include <stdio.h>
__global__ void body_k(double* x, int* it, cudaGraphConditionalHandle h, int kmax) {
    x[0] += 1.0; int i = ++it[0];
    cudaGraphSetConditional(h, i < kmax ? 1 : 0);
}
int main() {
    cudaGraph_t g; cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    printf("handle %d\n", (int)e);
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
    cudaGraphNode_t n; e = cudaGraphAddNode(&n, g, nullptr, 0, &p);
    printf("node %d\n", (int)e);
    cudaGraph_t body = p.conditional.phGraph_out[0];
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    double* x; int* it; cudaMalloc(&x, 8); cudaMalloc(&it, 4); cudaMemset(x, 0, 8); cudaMemset(it, 0, 4);
    e = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    printf("begin %d\n", (int)e);
    body_k<<<1,1,0,s>>>(x, it, h, 5);
    cudaGraph_t out; e = cudaStreamEndCapture(s, &out); printf("end %d\n", (int)e);
    cudaGraphExec_t ex; e = cudaGraphInstantiate(&ex, g, 0); printf("inst %d\n", (int)e);
    e = cudaGraphLaunch(ex, s); cudaStreamSynchronize(s); printf("launch %d\n", (int)e);
    double hx; int hit; cudaMemcpy(&hx, x, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&hit, it, 4, cudaMemcpyDeviceToHost);
    printf("x=%g it=%d\n", hx, hit);
    return 0;
}
