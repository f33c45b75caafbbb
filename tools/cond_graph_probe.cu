// Probe: nested conditional WHILE nodes driven from device code (CUDA 12.9, sm_100a).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_body(int* ctr, int* inner, cudaGraphConditionalHandle h_in) {
    inner[0] += 1;
    ctr[1] += 1;
    cudaGraphSetConditional(h_in, inner[0] < 3 ? 1 : 0);
}
__global__ void k_outer(int* ctr, int* inner, cudaGraphConditionalHandle h_out, cudaGraphConditionalHandle h_in) {
    cudaGraphSetConditional(h_in, 1);
    ctr[0] += 1;
    inner[0] = 0;
    cudaGraphSetConditional(h_out, ctr[0] < 4 ? 1 : 0);
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s -> %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

int probe2(int);
int probe1() {
    int *ctr, *inner;
    CK(cudaMalloc(&ctr, 8));
    CK(cudaMalloc(&inner, 4));
    CK(cudaMemset(ctr, 0, 8));
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h_out, h_in;
    CK(cudaGraphConditionalHandleCreate(&h_out, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h_out;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t n_out;
    CK(cudaGraphAddNode(&n_out, g, nullptr, 0, &p));
    cudaGraph_t body = p.conditional.phGraph_out[0];
    CK(cudaGraphConditionalHandleCreate(&h_in, body, 1, cudaGraphCondAssignDefault));
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    // outer body: capture k_outer, then an inner WHILE node
    CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    k_outer<<<1, 1, 0, s>>>(ctr, inner, h_out, h_in);
    cudaStreamCaptureStatus st;
    const cudaGraphNode_t* deps;
    size_t ndeps;
    cudaGraph_t cg;
    CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &ndeps));
    cudaGraphNodeParams pi = {};
    pi.type = cudaGraphNodeTypeConditional;
    pi.conditional.handle = h_in;
    pi.conditional.type = cudaGraphCondTypeWhile;
    pi.conditional.size = 1;
    cudaGraphNode_t n_in;
    CK(cudaGraphAddNode(&n_in, cg, deps, ndeps, &pi));
    CK(cudaStreamUpdateCaptureDependencies(s, &n_in, 1, cudaStreamSetCaptureDependencies));
    CK(cudaStreamEndCapture(s, &cg));
    cudaGraph_t ibody = pi.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(s, ibody, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    k_body<<<1, 1, 0, s>>>(ctr, inner, h_in);
    CK(cudaStreamEndCapture(s, &ibody));
    cudaGraphExec_t ex;
    CK(cudaGraphInstantiate(&ex, g, 0));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaMemsetAsync(ctr, 0, 8, s));
        cudaEventRecord(a, s);
        CK(cudaGraphLaunch(ex, s));
        cudaEventRecord(b, s);
        CK(cudaStreamSynchronize(s));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        int h[2];
        CK(cudaMemcpy(h, ctr, 8, cudaMemcpyDeviceToHost));
        printf("outer=%d inner_total=%d (expect 4, 12) time=%.1f us\n", h[0], h[1], ms * 1e3);
    }
    return 0;
}

// second probe: per-iteration overhead of a WHILE loop with N kernel nodes
__global__ void k_inc(int* c, cudaGraphConditionalHandle h, int limit, int last) {
    if (last) { c[0] += 1; cudaGraphSetConditional(h, c[0] < limit ? 1 : 0); }
}
int probe2(int nodes) {
    int* c;
    cudaMalloc(&c, 4);
    cudaGraph_t g;
    cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t n;
    cudaGraphAddNode(&n, g, nullptr, 0, &p);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaGraph_t body = p.conditional.phGraph_out[0];
    cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
    for (int i = 0; i < nodes; ++i) k_inc<<<148, 128, 0, s>>>(c, h, 1000, i == nodes - 1);
    cudaStreamEndCapture(s, &body);
    cudaGraphExec_t ex;
    if (cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) { printf("inst fail\n"); return 1; }
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemsetAsync(c, 0, 4, s);
        cudaEventRecord(a, s);
        cudaGraphLaunch(ex, s);
        cudaEventRecord(b, s);
        cudaStreamSynchronize(s);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("nodes/iter=%d: %.2f us per iteration, %.2f us per node\n", nodes, ms * 1e3 / 1000, ms * 1e3 / 1000 / nodes);
    }
    // plain stream launches for comparison
    cudaEventRecord(a, s);
    for (int i = 0; i < 1000 * nodes; ++i) k_inc<<<148, 128, 0, s>>>(c, h, 1000, 0);
    cudaEventRecord(b, s);
    cudaStreamSynchronize(s);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("stream launches: %.2f us per kernel\n", ms * 1e3 / 1000 / nodes);
    return 0;
}
int main() { probe1(); probe2(1); probe2(8); probe2(32); return 0; }
