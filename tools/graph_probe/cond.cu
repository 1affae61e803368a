#include <cstdio>
#include <cuda_runtime.h>
__global__ void body(int* ctr, cudaGraphConditionalHandle h, cudaGraphConditionalHandle h2) {
    __shared__ int last;
    if (threadIdx.x == 0) {
        int v = atomicAdd(&ctr[1], 1);
        last = (v == gridDim.x - 1);
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        ctr[1] = 0;
        int it = ++ctr[0];
        cudaGraphSetConditional(h, it < 10 ? 1 : 0);
        cudaGraphSetConditional(h2, (it % 2) ? 1 : 0);
    }
}
__global__ void odd(int* ctr) { if (threadIdx.x == 0 && blockIdx.x == 0) ctr[2] += 1; }
int main() {
    int* d; cudaMalloc(&d, 16); cudaMemset(d, 0, 16);
    cudaGraph_t g; cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h, h2;
    cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h; cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
    cudaGraphNode_t wn;
    cudaError_t e = cudaGraphAddNode(&wn, g, nullptr, 0, &cp);
    printf("add while: %s\n", cudaGetErrorString(e));
    cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
    cudaGraphConditionalHandleCreate(&h2, bodyg, 0, cudaGraphCondAssignDefault);
    cudaGraphNodeParams kp = {};
    kp.type = cudaGraphNodeTypeKernel;
    void* args[] = {&d, &h, &h2};
    kp.kernel.func = (void*)body; kp.kernel.gridDim = dim3(148); kp.kernel.blockDim = dim3(256); kp.kernel.kernelParams = args;
    cudaGraphNode_t kn; e = cudaGraphAddNode(&kn, bodyg, nullptr, 0, &kp); printf("add body: %s\n", cudaGetErrorString(e));
    cudaGraphNodeParams ip = {}; ip.type = cudaGraphNodeTypeConditional; ip.conditional.handle = h2; ip.conditional.type = cudaGraphCondTypeIf; ip.conditional.size = 1;
    cudaGraphNode_t in; e = cudaGraphAddNode(&in, bodyg, &kn, 1, &ip); printf("add if: %s\n", cudaGetErrorString(e));
    cudaGraphNodeParams op = {}; op.type = cudaGraphNodeTypeKernel; void* a2[] = {&d};
    op.kernel.func = (void*)odd; op.kernel.gridDim = dim3(1); op.kernel.blockDim = dim3(32); op.kernel.kernelParams = a2;
    cudaGraphNode_t on; e = cudaGraphAddNode(&on, ip.conditional.phGraph_out[0], nullptr, 0, &op); printf("add odd: %s\n", cudaGetErrorString(e));
    cudaGraphExec_t x; e = cudaGraphInstantiate(&x, g, 0); printf("inst: %s\n", cudaGetErrorString(e));
    cudaStream_t s; cudaStreamCreate(&s);
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(d, 0, 16);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a, s);
        e = cudaGraphLaunch(x, s);
        cudaEventRecord(b, s);
        cudaStreamSynchronize(s);
        float ms; cudaEventElapsedTime(&ms, a, b);
        int hd[4]; cudaMemcpy(hd, d, 16, cudaMemcpyDeviceToHost);
        printf("launch %s iters=%d odd=%d time=%.1f us (%.2f us/iter)\n", cudaGetErrorString(e), hd[0], hd[2], ms*1e3, ms*1e3/ hd[0]);
    }
    return 0;
}
