// Microbenchmark: scattered fp32 row accumulation into global memory on sm_100a.
//   mode 0: red.global.add.v4.f32 from registers (one thread per row, C/4 instructions)
//   mode 1: rows staged in smem, one cp.reduce.async.bulk .add.f32 per row (TMA engine)
// 148 CTAs x 128 threads; each CTA accumulates `rows` random rows of C floats per iteration.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/red_bench.cu -o scripts/red_bench.bin
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

template <int C, int MODE>
__global__ void __launch_bounds__(128) k(float *__restrict__ acc, const int *__restrict__ idx, int n_rows, int iters) {
    __shared__ __align__(128) float stage[MODE == 1 ? 128 * C : 4];
    const int t = threadIdx.x;
    if (MODE == 1) for (int i = t; i < 128 * C; i += 128) stage[i] = 1.0f;
    __syncthreads();
    for (int it = 0; it < iters; ++it) {
        const int row = idx[((blockIdx.x * iters + it) * 128 + t) % (1 << 20)] % n_rows;
        float *dst = acc + (size_t)row * C;
        if (MODE == 0) {
#pragma unroll
            for (int c = 0; c < C; c += 4)
                asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(dst + c), "f"(1.f), "f"(1.f), "f"(1.f),
                             "f"(1.f)
                             : "memory");
        } else {
            const uint32_t src = (uint32_t)__cvta_generic_to_shared(stage + t * C);
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
                         "r"(src), "r"(C * 4)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if ((it & 7) == 7) asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
        }
    }
    if (MODE == 1) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int C, int MODE>
void run(float *acc, const int *idx, int n_rows) {
    const int iters = 400;
    k<C, MODE><<<148, 128>>>(acc, idx, n_rows, iters);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<C, MODE><<<148, 128>>>(acc, idx, n_rows, iters);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = 148.0 * 128 * iters * C * 4;
    printf("C=%3d mode=%d (%s): %8.1f us  %7.2f TB/s of fp32 reduced %s\n", C, MODE,
           MODE == 0 ? "red.v4 per thread" : "bulk reduce per row", ms * 1e3, bytes / (ms * 1e-3) / 1e12,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    const int n_rows = 100000;
    float *acc;
    int *idx;
    cudaMalloc(&acc, (size_t)n_rows * 256 * 4);
    cudaMemset(acc, 0, (size_t)n_rows * 256 * 4);
    cudaMalloc(&idx, (1 << 20) * 4);
    std::vector<int> h(1 << 20);
    srand(2);
    for (auto &v : h) v = rand();
    cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    run<32, 0>(acc, idx, n_rows);
    run<32, 1>(acc, idx, n_rows);
    run<96, 0>(acc, idx, n_rows);
    run<96, 1>(acc, idx, n_rows);
    run<64, 0>(acc, idx, n_rows);
    run<64, 1>(acc, idx, n_rows);
    run<64, 0>(acc, idx, 7000);      // a level-3-sized accumulator (hot rows)
    run<64, 1>(acc, idx, 7000);
    run<256, 0>(acc, idx, 7000);
    run<256, 0>(acc, idx, n_rows);
    return 0;
}
