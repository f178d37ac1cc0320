// Cost of the BFS device loop's graph machinery on B200: a WHILE node whose
// body is `decide` (one-warp kernel setting a SWITCH handle) -> SWITCH with
// one body of K empty kernels; per-iteration time vs K.  Also: the same
// K kernels in a plain captured graph (no conditionals), and a body kernel
// that runs L "levels" internally (what a single-CTA tail loop would pay).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o graph_cond_mb graph_cond_mb.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void decide(int* it, int iters, int sel, cudaGraphConditionalHandle hs, cudaGraphConditionalHandle hw) {
    if (threadIdx.x) return;
    int i = ++*it;
    cudaGraphSetConditional(hs, sel);
    if (i >= iters) cudaGraphSetConditional(hw, 0);
}
__global__ void work(int* sink) { if (threadIdx.x == 0 && blockIdx.x == 0 && *sink == 12345) *sink = 0; }

int run(int K, int iters, unsigned grid, float* us) {
    cudaStream_t s, s2;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    int* it; int* sink;
    CK(cudaMalloc(&it, 4)); CK(cudaMalloc(&sink, 4)); CK(cudaMemset(sink, 0, 4));
    cudaGraph_t g; CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle hw, hs;
    CK(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
    CK(cudaGraphConditionalHandleCreate(&hs, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams wp{}; wp.type = cudaGraphNodeTypeConditional; wp.conditional.handle = hw;
    wp.conditional.type = cudaGraphCondTypeWhile; wp.conditional.size = 1;
    cudaGraphNode_t wn; CK(cudaGraphAddNode(&wn, g, nullptr, 0, &wp));
    cudaGraph_t body = wp.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    decide<<<1, 32, 0, s>>>(it, iters, K == 0 ? 7 : 0, hs, hw);
    {
        cudaStreamCaptureStatus cs; cudaGraph_t cg; const cudaGraphNode_t* deps; size_t nd;
        CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &cg, &deps, &nd));
        cudaGraphNodeParams ip{}; ip.type = cudaGraphNodeTypeConditional; ip.conditional.handle = hs;
        ip.conditional.type = cudaGraphCondTypeSwitch; ip.conditional.size = 2;
        cudaGraphNode_t node; CK(cudaGraphAddNode(&node, cg, deps, nd, &ip));
        CK(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
        for (int b = 0; b < 2; ++b) {
            cudaGraph_t bg = ip.conditional.phGraph_out[b];
            CK(cudaStreamBeginCaptureToGraph(s2, bg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
            for (int k = 0; k < (b == 0 ? (K > 0 ? K : 1) : 1); ++k) work<<<grid, 256, 0, s2>>>(sink);
            CK(cudaStreamEndCapture(s2, &bg));
        }
    }
    CK(cudaStreamEndCapture(s, &body));
    cudaGraphExec_t ex; CK(cudaGraphInstantiate(&ex, g, 0));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CK(cudaMemsetAsync(it, 0, 4, s));
        CK(cudaEventRecord(a, s));
        CK(cudaGraphLaunch(ex, s));
        CK(cudaEventRecord(b, s));
        CK(cudaStreamSynchronize(s));
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    *us = best * 1000.f;
    return 0;
}

int main() {
    const int iters = 200;
    for (unsigned grid : {1u, 148u, 1184u, 16384u}) {
        for (int K : {0, 1, 2, 3, 5}) {
            float us;
            if (run(K, iters, grid, &us)) return 1;
            printf("grid %5u  WHILE{decide -> SWITCH{%d kernels (0: no body selected)}}: %.2f us/iter\n", grid, K, us / iters);
        }
    }
    return 0;
}
