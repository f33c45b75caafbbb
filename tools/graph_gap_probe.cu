// Probe: node-to-node latency of kernel chains inside a captured CUDA graph on
// sm_100a, with and without programmatic dependent launch (PDL), at top level
// and inside a conditional WHILE body (the shape of the engine's Newton loop),
// and the cost of an IF node in the middle of that body (mode `if0` / `if1`:
// the IF's condition false / true, its body one kernel).
// Each kernel is a small grid that does a few dependent global updates, so
// the measured time per node is launch/dependency latency, not work.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gap tools/graph_gap_probe.cu && /tmp/gap
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                                     \
    do {                                                                                          \
        cudaError_t e = (x);                                                                      \
        if (e != cudaSuccess) {                                                                   \
            printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));            \
            return 1;                                                                             \
        }                                                                                         \
    } while (0)

__global__ void k_step(double* buf, int n, int pdl) {
    if (pdl) {
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) buf[i] = buf[i] * 0.5 + 1.0;
}

__global__ void k_ctrl(int* ctr, int iters, cudaGraphConditionalHandle h) {
    const int c = ++ctr[0];
    cudaGraphSetConditional(h, c < iters ? 1 : 0);
}

__global__ void k_ctrl2(int* ctr, int iters, cudaGraphConditionalHandle h, cudaGraphConditionalHandle h2,
                        int ifval) {
    const int c = ++ctr[0];
    cudaGraphSetConditional(h, c < iters ? 1 : 0);
    cudaGraphSetConditional(h2, ifval ? 1u : 0u);
}

static int launch(double* buf, int n, int blocks, bool pdl, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, k_step, buf, n, pdl ? 1 : 0));
    return 0;
}

// chain of `len` kernels, repeated `reps` times at top level
static int top_level(double* buf, int n, int blocks, int len, bool pdl, float* us_per_node) {
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int k = 0; k < len; ++k)
        if (launch(buf, n, blocks, pdl, s)) return 1;
    CK(cudaStreamEndCapture(s, &g));
    cudaGraphExec_t ge;
    CK(cudaGraphInstantiate(&ge, g, 0));
    for (int w = 0; w < 3; ++w) CK(cudaGraphLaunch(ge, s));
    CK(cudaStreamSynchronize(s));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const int reps = 20;
    CK(cudaEventRecord(a, s));
    for (int r = 0; r < reps; ++r) CK(cudaGraphLaunch(ge, s));
    CK(cudaEventRecord(b, s));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    *us_per_node = 1000.f * ms / (reps * len);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaStreamDestroy(s);
    return 0;
}

// WHILE(iters) { k_ctrl; `len` kernels } inside one graph
static int in_while(double* buf, int n, int blocks, int len, int iters, bool pdl, float* us_per_iter) {
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    int* ctr;
    CK(cudaMalloc(&ctr, sizeof(int)));
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, g, nullptr, 0, &p));
    cudaGraph_t body = p.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    k_ctrl<<<1, 1, 0, s>>>(ctr, iters, h);
    for (int k = 0; k < len; ++k)
        if (launch(buf, n, blocks, pdl, s)) return 1;
    CK(cudaStreamEndCapture(s, nullptr));
    cudaGraphExec_t ge;
    CK(cudaGraphInstantiate(&ge, g, 0));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int w = 0; w < 2; ++w) {
        CK(cudaMemsetAsync(ctr, 0, sizeof(int), s));
        CK(cudaGraphLaunch(ge, s));
    }
    CK(cudaStreamSynchronize(s));
    CK(cudaMemsetAsync(ctr, 0, sizeof(int), s));
    CK(cudaEventRecord(a, s));
    CK(cudaGraphLaunch(ge, s));
    CK(cudaEventRecord(b, s));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    *us_per_iter = 1000.f * ms / iters;
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaFree(ctr);
    cudaStreamDestroy(s);
    return 0;
}

// WHILE(iters) { k_ctrl2; 4 kernels; IF(ifval) { 1 kernel }; 4 kernels }
static int in_while_if(double* buf, int n, int blocks, int iters, int ifval, float* us_per_iter) {
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    int* ctr;
    CK(cudaMalloc(&ctr, sizeof(int)));
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, g, nullptr, 0, &p));
    cudaGraph_t body = p.conditional.phGraph_out[0];
    cudaGraphConditionalHandle h2;
    CK(cudaGraphConditionalHandleCreate(&h2, body, 0, 0));
    CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    k_ctrl2<<<1, 1, 0, s>>>(ctr, iters, h, h2, ifval);
    for (int k = 0; k < 4; ++k)
        if (launch(buf, n, blocks, false, s)) return 1;
    {
        cudaStreamCaptureStatus st;
        cudaGraph_t cg;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &nd));
        cudaGraphNodeParams q = {};
        q.type = cudaGraphNodeTypeConditional;
        q.conditional.handle = h2;
        q.conditional.type = cudaGraphCondTypeIf;
        q.conditional.size = 1;
        cudaGraphNode_t ifn;
        CK(cudaGraphAddNode(&ifn, cg, deps, nd, &q));
        CK(cudaStreamUpdateCaptureDependencies(s, &ifn, 1, cudaStreamSetCaptureDependencies));
        cudaStream_t s2;
        CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        CK(cudaStreamBeginCaptureToGraph(s2, q.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                         cudaStreamCaptureModeRelaxed));
        if (launch(buf, n, blocks, false, s2)) return 1;
        CK(cudaStreamEndCapture(s2, nullptr));
    }
    for (int k = 0; k < 4; ++k)
        if (launch(buf, n, blocks, false, s)) return 1;
    CK(cudaStreamEndCapture(s, nullptr));
    cudaGraphExec_t ge;
    CK(cudaGraphInstantiate(&ge, g, 0));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int w = 0; w < 2; ++w) {
        CK(cudaMemsetAsync(ctr, 0, sizeof(int), s));
        CK(cudaGraphLaunch(ge, s));
    }
    CK(cudaStreamSynchronize(s));
    CK(cudaMemsetAsync(ctr, 0, sizeof(int), s));
    CK(cudaEventRecord(a, s));
    CK(cudaGraphLaunch(ge, s));
    CK(cudaEventRecord(b, s));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    *us_per_iter = 1000.f * ms / iters;
    return 0;
}

// usage: gap <blocks> <pdl 0|1> <mode: top|while|if0|if1>
int main(int argc, char** argv) {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const int blocks = argc > 1 ? atoi(argv[1]) : 148;
    const int pdl = argc > 2 ? atoi(argv[2]) : 0;
    const bool top = argc <= 3 || argv[3][0] == 't';
    const int n = blocks * 256;
    double* buf;
    CK(cudaMalloc(&buf, n * sizeof(double)));
    CK(cudaMemset(buf, 0, n * sizeof(double)));
    float t = 0.f;
    if (argc > 3 && argv[3][0] == 'i') {
        const int ifval = argv[3][2] == '1';
        if (in_while_if(buf, n, blocks, 200, ifval, &t)) return 1;
        printf("{\"blocks\": %d, \"if\": %d, \"while_us_per_iter_ctrl_plus_8_plus_if\": %.3f}\n", blocks, ifval, t);
    } else if (top) {
        if (top_level(buf, n, blocks, 16, pdl, &t)) return 1;
        printf("{\"blocks\": %d, \"pdl\": %d, \"top_level_us_per_node\": %.3f}\n", blocks, pdl, t);
    } else {
        if (in_while(buf, n, blocks, 8, 200, pdl, &t)) return 1;
        printf("{\"blocks\": %d, \"pdl\": %d, \"while_us_per_iter_ctrl_plus_8\": %.3f, \"per_kernel\": %.3f}\n",
               blocks, pdl, t, t / 9.0);
    }
    return 0;
}
