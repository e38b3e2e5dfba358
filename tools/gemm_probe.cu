// standalone timing of tc_gemm_kernel (the learner's tcgen05 GEMM) in isolation
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <vector>
#include "../paper_2111_05188_b200/csrc/gemm_kernel.cuh"  // nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/gp tools/gemm_probe.cu
using namespace pod;
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn enc;
static int g_pdl = 0;  // 1: launches carry the PDL attribute (the kernel itself no longer waits)
static void mk(CUtensorMap* m, void* p, uint64_t K, uint64_t rows, uint64_t ld, uint32_t brow) {
    cuuint64_t d[2] = {K, rows}, s[1] = {ld * 2};
    cuuint32_t b[2] = {64, brow}, e[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) printf("encode failed %d\n", r);
}
template <int BN>
void run(int M, int N, int K, int mode, const char* name) {
    __nv_bfloat16 *A, *B, *O, *OT, *XL; float *bias, *outf, *bp;
    cudaMalloc(&A, (size_t)M * K * 2); cudaMalloc(&B, (size_t)N * K * 2);
    cudaMalloc(&O, (size_t)M * N * 2); cudaMalloc(&OT, (size_t)M * N * 2); cudaMalloc(&XL, (size_t)M * N * 2);
    cudaMalloc(&bias, N * 4); cudaMalloc(&outf, (size_t)M * N * 4); cudaMalloc(&bp, (size_t)M * N * 4);
    cudaMemset(A, 0, (size_t)M * K * 2); cudaMemset(B, 0, (size_t)N * K * 2); cudaMemset(bias, 0, N * 4); cudaMemset(XL, 0, (size_t)M*N*2);
    CUtensorMap ma, mb;
    mk(&ma, A, K, M, K, 128); mk(&mb, B, K, N, K, BN);
    GemmEpi<__nv_bfloat16> ep{};
    ep.mode = mode; ep.M = M; ep.N = N; ep.act = 0; ep.bias = bias; ep.out = O; ep.out_t = OT; ep.outf = outf;
    ep.xl = XL; ep.bpart = bp; ep.ld_out = N; ep.ld_out_t = M; ep.ld_outf = N; ep.ld_xl = N;
    cudaFuncSetAttribute(tc_gemm_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm_smem_bytes(BN));
    dim3 grid(M / 128, (N + BN - 1) / BN);
    for (int i = 0; i < 3; ++i) tc_gemm_kernel<BN><<<grid, 128, gemm_smem_bytes(BN)>>>(ma, mb, ep, K);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int reps = 50;
    cudaStream_t cs; cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < reps; ++i) {
        cudaLaunchConfig_t lc{}; lc.gridDim = grid; lc.blockDim = dim3(128); lc.dynamicSmemBytes = gemm_smem_bytes(BN); lc.stream = cs;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = g_pdl; lc.attrs = at; lc.numAttrs = 1;
        cudaLaunchKernelEx(&lc, tc_gemm_kernel<BN>, ma, mb, ep, K);
    }
    cudaStreamEndCapture(cs, &g); cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, cs); cudaStreamSynchronize(cs);
    cudaEventRecord(e0, cs);
    cudaGraphLaunch(ge, cs);
    cudaEventRecord(e1, cs); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    double us = ms * 1e3 / reps;
    printf("%-10s BN=%3d M=%5d N=%4d K=%5d grid=%3d: %7.2f us/launch  %6.1f TFLOP/s %s\n", name, BN, M, N, K,
           grid.x * grid.y, us, 2.0 * M * N * K / (us * 1e-6) / 1e12, err ? cudaGetErrorString(err) : "");
    cudaFree(A); cudaFree(B); cudaFree(O); cudaFree(OT); cudaFree(XL); cudaFree(bias); cudaFree(outf); cudaFree(bp);
}
__global__ void empty_kernel(int x) { if (x == 12345) printf("x"); }
int main() {
    cudaDriverEntryPointQueryResult q; void* p;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q); enc = (EncodeTiledFn)p;
    {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int i = 0; i < 10; ++i) empty_kernel<<<64, 128>>>(1);
        cudaEventRecord(e0);
        for (int i = 0; i < 50; ++i) empty_kernel<<<64, 128>>>(1);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("empty kernel: %.2f us/launch\n", ms * 1e3 / 50);
    }
    for (int pdl : {0, 1}) {
    g_pdl = pdl;
    printf("graph, pdl=%d\n", pdl);
    for (int K : {64, 128, 256}) run<64>(1024, 512, K, 2, "dW-K");
    for (int mode : {0, 2, 3}) {
        const char* nm = mode == 0 ? "fwd" : mode == 2 ? "dW" : "dX";
        int M = mode == 2 ? 512 : 1024, K = mode == 2 ? 1024 : 512;
        run<64>(M, 512, K, mode, nm);
        run<128>(M, 512, K, mode, nm);
        run<32>(M, 512, K, mode, nm);
    }
    run<64>(8192, 512, 512, 0, "fwd-big");
    run<128>(8192, 512, 512, 0, "fwd-big");
    }
}
