#include <cuda_runtime.h>
#include <cstdio>
__global__ void setc(cudaGraphConditionalHandle h, int* ctr, int limit) {
    int v = ++(*ctr);
    cudaGraphSetConditional(h, v < limit ? 1 : 0);
}
__global__ void body(int* x) { atomicAdd(x, 1); }
int main() {
    int *ctr, *x;
    cudaMalloc(&ctr, 4); cudaMalloc(&x, 4); cudaMemset(ctr, 0, 4); cudaMemset(x, 0, 4);
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaGraph_t g; cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    printf("handle %s\n", cudaGetErrorString(e));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
    cudaGraphNode_t node;
    e = cudaGraphAddNode(&node, g, nullptr, 0, &p);
    printf("add %s\n", cudaGetErrorString(e));
    cudaGraph_t bodyg = p.conditional.phGraph_out[0];
    e = cudaStreamBeginCaptureToGraph(s, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
    printf("cap %s\n", cudaGetErrorString(e));
    body<<<1, 32, 0, s>>>(x);
    setc<<<1, 1, 0, s>>>(h, ctr, 100);
    e = cudaStreamEndCapture(s, &bodyg);
    printf("end %s\n", cudaGetErrorString(e));
    cudaGraphExec_t ex; e = cudaGraphInstantiate(&ex, g, 0);
    printf("inst %s\n", cudaGetErrorString(e));
    e = cudaGraphLaunch(ex, s); cudaStreamSynchronize(s);
    int hx; cudaMemcpy(&hx, x, 4, cudaMemcpyDeviceToHost);
    printf("launch %s x=%d (expect 3200)\n", cudaGetErrorString(e), hx);
    return 0;
}
