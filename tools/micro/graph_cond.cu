// Feasibility probe: a WHILE conditional node whose body is stream-captured kernels
// launched with programmatic stream serialization, condition set from device code.
#include <cuda_runtime.h>
#include <cstdio>
__global__ void k_work(int *ctr, int *log) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0) { int i = atomicAdd(ctr, 1); log[i] = i; }
}
__global__ void k_cond(cudaGraphConditionalHandle h, int *ctr, int limit) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    cudaGraphSetConditional(h, *ctr < limit ? 1u : 0u);
}
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 g, dim3 b, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g; cfg.blockDim = b; cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...);
}
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
int main() {
    int *ctr, *log;
    CK(cudaMalloc(&ctr, 4)); CK(cudaMalloc(&log, 4096));
    cudaStream_t st; CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaGraph_t g; CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h; cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
    cudaGraphNode_t cn; CK(cudaGraphAddNode(&cn, g, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    for (int i = 0; i < 3; ++i) CK(launch_pdl(k_work, 4, 64, st, ctr, log));
    CK(launch_pdl(k_cond, 1, 1, st, h, ctr, 30));
    CK(cudaStreamEndCapture(st, &body));
    cudaGraphExec_t ex; CK(cudaGraphInstantiate(&ex, g, 0));
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaMemsetAsync(ctr, 0, 4, st));
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a, st);
        CK(cudaGraphLaunch(ex, st));
        cudaEventRecord(b, st);
        CK(cudaStreamSynchronize(st));
        float ms; cudaEventElapsedTime(&ms, a, b);
        int hc; CK(cudaMemcpy(&hc, ctr, 4, cudaMemcpyDeviceToHost));
        printf("rep %d: ctr=%d (want 30) %.3f ms\n", rep, hc, ms);
    }
    // a graph whose first batch is launched directly, then the while graph with condition default 0 set by a kernel
    printf("graph_cond OK\n");
    return 0;
}
