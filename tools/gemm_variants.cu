// gemm_variants.cu — K1 main-loop variants timed side by side (tuning tool, not
// product code).  D = C − A·B (A M×K, B K×N row-major FP64) on DMMA.8x8x4 with
// the production epilogue shape; cuBLAS DGEMM on the same operands for scale.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//        tools/gemm_variants.cu -lcublas -o gemm_variants && ./gemm_variants
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e_ = (x);                                                  \
        if (e_ != cudaSuccess) {                                               \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                           \
        }                                                                      \
    } while (0)

__device__ __forceinline__ void cp_async16(double* smem, const double* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// WM×WN warps, warp tile (FM·8)×(FN·8); CTA tile BM×BN = (WM·FM·8)×(WN·FN·8)
template <int WM, int WN, int FM, int FN, int BK, int STAGES, bool DB, int MINB>
struct Cfg {
    static constexpr int BM = WM * FM * 8, BN = WN * FN * 8, THREADS = WM * WN * 32;
    static constexpr int PAD = 4, A_LD = BK + PAD, B_LD = BN + PAD;
    static constexpr int A_STAGE = BM * A_LD, B_STAGE = BK * B_LD;
    static constexpr size_t SMEM = sizeof(double) * STAGES * (A_STAGE + B_STAGE);
};

template <class CF>
__device__ __forceinline__ void load_stage(const double* A, const double* B, long long K,
                                           long long N, double* As, double* Bs, long long m0,
                                           long long n0, long long k0) {
    const int tid = threadIdx.x;
    constexpr int AV = CF::BM * CF::A_LD;  (void)AV;
    constexpr int ACH = CF::BM * (CF::A_LD - CF::PAD) / 2;  // double2 chunks of A
#pragma unroll
    for (int e = tid; e < ACH; e += CF::THREADS) {
        constexpr int per_row = (CF::A_LD - CF::PAD) / 2;
        const int r = e / per_row, c2 = (e % per_row) * 2;
        cp_async16(As + r * CF::A_LD + c2, A + (m0 + r) * K + k0 + c2);
    }
    constexpr int BCH = (CF::B_LD - CF::PAD) / 2 * (CF::B_STAGE / CF::B_LD);
#pragma unroll
    for (int e = tid; e < BCH; e += CF::THREADS) {
        constexpr int per_row = (CF::B_LD - CF::PAD) / 2;
        const int r = e / per_row, c2 = (e % per_row) * 2;
        cp_async16(Bs + r * CF::B_LD + c2, B + (k0 + r) * N + n0 + c2);
    }
}

template <int WM, int WN, int FM, int FN, int BK, int STAGES, bool DB, int MINB>
__global__ void __launch_bounds__(WM* WN * 32, MINB)
    k_var(const double* __restrict__ A, const double* __restrict__ B, const double* __restrict__ Cin,
          double* __restrict__ D, long long M, long long N, long long K, double* part) {
    using CF = Cfg<WM, WN, FM, FN, BK, STAGES, DB, MINB>;
    extern __shared__ __align__(16) double sm[];
    double* As = sm;
    double* Bs = sm + STAGES * CF::A_STAGE;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const int gq = lane >> 2, tq = lane & 3;
    const long long m0 = (long long)blockIdx.y * CF::BM, n0 = (long long)blockIdx.x * CF::BN;
    const long long KT = K / BK;
    double acc[FM][FN][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < KT) load_stage<CF>(A, B, K, N, As + s * CF::A_STAGE, Bs + s * CF::B_STAGE, m0, n0, s * BK);
        cp_commit();
    }
    for (long long kt = 0; kt < KT; ++kt) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        const long long nk = kt + STAGES - 1;
        if (nk < KT) {
            const int st = (int)(nk % STAGES);
            load_stage<CF>(A, B, K, N, As + st * CF::A_STAGE, Bs + st * CF::B_STAGE, m0, n0, nk * BK);
        }
        cp_commit();
        const int cs = (int)(kt % STAGES);
        const double* a_s = As + cs * CF::A_STAGE + (wm * FM * 8 + gq) * CF::A_LD + tq;
        const double* b_s = Bs + cs * CF::B_STAGE + tq * CF::B_LD + wn * FN * 8 + gq;
        if (DB) {
            double af[2][FM], bf[2][FN];
#pragma unroll
            for (int mi = 0; mi < FM; ++mi) af[0][mi] = a_s[mi * 8 * CF::A_LD];
#pragma unroll
            for (int ni = 0; ni < FN; ++ni) bf[0][ni] = b_s[ni * 8];
#pragma unroll
            for (int kk = 0; kk < BK / 4; ++kk) {
                const int cur = kk & 1, nxt = cur ^ 1;
                if (kk + 1 < BK / 4) {
#pragma unroll
                    for (int mi = 0; mi < FM; ++mi) af[nxt][mi] = a_s[mi * 8 * CF::A_LD + (kk + 1) * 4];
#pragma unroll
                    for (int ni = 0; ni < FN; ++ni) bf[nxt][ni] = b_s[(kk + 1) * 4 * CF::B_LD + ni * 8];
                }
#pragma unroll
                for (int mi = 0; mi < FM; ++mi)
#pragma unroll
                    for (int ni = 0; ni < FN; ++ni)
                        dmma(acc[mi][ni][0], acc[mi][ni][1], af[cur][mi], bf[cur][ni]);
            }
        } else {
#pragma unroll
            for (int kk = 0; kk < BK / 4; ++kk) {
                double af[FM], bf[FN];
#pragma unroll
                for (int mi = 0; mi < FM; ++mi) af[mi] = a_s[mi * 8 * CF::A_LD + kk * 4];
#pragma unroll
                for (int ni = 0; ni < FN; ++ni) bf[ni] = b_s[kk * 4 * CF::B_LD + ni * 8];
#pragma unroll
                for (int mi = 0; mi < FM; ++mi)
#pragma unroll
                    for (int ni = 0; ni < FN; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
            }
        }
    }
    cp_wait<0>();
    double sq = 0.0;
#pragma unroll
    for (int mi = 0; mi < FM; ++mi) {
        const long long r = m0 + wm * FM * 8 + mi * 8 + gq;
#pragma unroll
        for (int ni = 0; ni < FN; ++ni) {
            const long long c = n0 + wn * FN * 8 + ni * 8 + 2 * tq;
            const double2 cc = *reinterpret_cast<const double2*>(Cin + r * N + c);
            const double o0 = cc.x - acc[mi][ni][0], o1 = cc.y - acc[mi][ni][1];
            sq += o0 * o0 + o1 * o1;
            *reinterpret_cast<double2*>(D + r * N + c) = make_double2(o0, o1);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if (lane == 0) atomicAdd(part, sq);
}

template <int WM, int WN, int FM, int FN, int BK, int STAGES, bool DB, int MINB>
float run(const char* name, const double* A, const double* B, const double* Cin, double* D,
          long long M, long long N, long long K, double* part, const double* Dref, int reps) {
    using CF = Cfg<WM, WN, FM, FN, BK, STAGES, DB, MINB>;
    auto kern = k_var<WM, WN, FM, FN, BK, STAGES, DB, MINB>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM));
    dim3 grid((unsigned)(N / CF::BN), (unsigned)(M / CF::BM));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<grid, CF::THREADS, CF::SMEM>>>(A, B, Cin, D, M, N, K, part);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) kern<<<grid, CF::THREADS, CF::SMEM>>>(A, B, Cin, D, M, N, K, part);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    // check against the cuBLAS result on a sample
    std::vector<double> h(4096), hr(4096);
    CK(cudaMemcpy(h.data(), D, sizeof(double) * 4096, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hr.data(), Dref, sizeof(double) * 4096, cudaMemcpyDeviceToHost));
    double err = 0, nrm = 0;
    for (int i = 0; i < 4096; ++i) {
        err = fmax(err, fabs(h[i] - hr[i]));
        nrm = fmax(nrm, fabs(hr[i]));
    }
    int regs = 0;
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess) regs = fa.numRegs;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, CF::THREADS, CF::SMEM);
    printf("%-34s tile %3dx%3d BK %2d st %d regs %3d cta/sm %d smem %6zu: %8.3f ms %6.2f TFLOP/s  maxerr %.2e\n",
           name, CF::BM, CF::BN, BK, STAGES, regs, occ, CF::SMEM, ms, 2.0 * M * N * K / ms / 1e9,
           err / nrm);
    return ms;
}

int main(int argc, char** argv) {
    long long M = 8192, N = 8192, K = 2048;
    if (argc > 3) {
        M = atoll(argv[1]);
        N = atoll(argv[2]);
        K = atoll(argv[3]);
    }
    const int reps = argc > 4 ? atoi(argv[4]) : 5;
    double *A, *B, *Cin, *D, *Dref, *part;
    CK(cudaMalloc(&A, sizeof(double) * M * K));
    CK(cudaMalloc(&B, sizeof(double) * K * N));
    CK(cudaMalloc(&Cin, sizeof(double) * M * N));
    CK(cudaMalloc(&D, sizeof(double) * M * N));
    CK(cudaMalloc(&Dref, sizeof(double) * M * N));
    CK(cudaMalloc(&part, sizeof(double)));
    {
        std::vector<double> h(std::max(M * K, K * N));
        unsigned long long s = 88172645463325252ull;
        for (auto& v : h) {
            s ^= s << 13; s ^= s >> 7; s ^= s << 17;
            v = (double)(s >> 11) * 0x1.0p-53 - 0.5;
        }
        CK(cudaMemcpy(A, h.data(), sizeof(double) * M * K, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(B, h.data(), sizeof(double) * K * N, cudaMemcpyHostToDevice));
        CK(cudaMemset(Cin, 0, sizeof(double) * M * N));
    }
    cublasHandle_t hb;
    cublasCreate(&hb);
    const double one = 1.0, mone = -1.0;
    // row-major D = 0 − A·B  ⇔ column-major Dᵀ = −Bᵀ·Aᵀ
    CK(cudaMemcpy(Dref, Cin, sizeof(double) * M * N, cudaMemcpyDeviceToDevice));
    cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, (int)N, (int)M, (int)K, &mone, B, (int)N, A, (int)K, &one, Dref, (int)N);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r)
        cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, (int)N, (int)M, (int)K, &mone, B, (int)N, A, (int)K, &one, D, (int)N);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("M %lld N %lld K %lld\n%-34s %8.3f ms %6.2f TFLOP/s\n", M, N, K, "cuBLAS DGEMM", ms, 2.0 * M * N * K / ms / 1e9);

    run<2, 4, 8, 4, 16, 3, false, 1>("base 2x4 w64x32 BK16 S3", A, B, Cin, D, M, N, K, part, Dref, reps);
    run<2, 4, 8, 4, 16, 3, true, 1>("base+DB", A, B, Cin, D, M, N, K, part, Dref, reps);
    run<2, 4, 8, 4, 16, 4, false, 1>("S4", A, B, Cin, D, M, N, K, part, Dref, reps);
    run<2, 4, 8, 4, 32, 3, false, 1>("BK32 S3", A, B, Cin, D, M, N, K, part, Dref, reps);
    run<2, 4, 8, 4, 32, 3, true, 1>("BK32 S3 DB", A, B, Cin, D, M, N, K, part, Dref, reps);
    run<2, 2, 8, 4, 16, 3, false, 2>("2x2 w64x32 (128x64) 2cta", A, B, Cin, D, M, N, K, part, Dref, reps);
    run<2, 2, 8, 4, 16, 4, true, 2>("2x2 128x64 S4 DB 2cta", A, B, Cin, D, M, N, K, part, Dref, reps);
    run<2, 2, 4, 8, 16, 3, false, 2>("2x2 w32x64 (64x128) 2cta", A, B, Cin, D, M, N, K, part, Dref, reps);
    run<4, 4, 4, 4, 16, 3, false, 1>("4x4 w32x32 (128x128) 16 warps", A, B, Cin, D, M, N, K, part, Dref, reps);
    run<4, 4, 4, 4, 16, 4, true, 1>("4x4 w32x32 S4 DB", A, B, Cin, D, M, N, K, part, Dref, reps);
    run<4, 2, 4, 8, 16, 3, false, 1>("4x2 w32x64 (128x128)", A, B, Cin, D, M, N, K, part, Dref, reps);
    run<2, 4, 8, 4, 8, 4, false, 1>("BK8 S4", A, B, Cin, D, M, N, K, part, Dref, reps);
    return 0;
}
