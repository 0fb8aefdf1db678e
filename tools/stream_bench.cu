// Achievable HBM bandwidth for multi-stream elementwise kernels on this GPU:
// NR arrays read + NW arrays written per element (double2 vectorised), the
// access mix of the PCG iteration kernel (reads r, q, p, x, s, Dinv; writes r,
// p, q, x).  nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/stream_bench.cu -o /tmp/sb
#include <cstdio>
#include <cuda_runtime.h>

template <int NR, int NW>
__global__ void k(const double2 *const *in, double2 *const *out, long n2) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int a = 0; a < NR; ++a) {
      const double2 v = __ldcs(&in[a][i]);
      acc.x += v.x;
      acc.y += v.y;
    }
#pragma unroll
    for (int b = 0; b < NW; ++b) __stcs(&out[b][i], make_double2(acc.x + b, acc.y - b));
  }
}

template <int NR, int NW>
void run(double2 **d_in, double2 **d_out, long n2) {
  double2 **in_dev, **out_dev;
  cudaMalloc(&in_dev, sizeof(void *) * 8);
  cudaMalloc(&out_dev, sizeof(void *) * 8);
  cudaMemcpy(in_dev, d_in, sizeof(void *) * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(out_dev, d_out, sizeof(void *) * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k<NR, NW><<<148 * 8, 256>>>(in_dev, out_dev, n2);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int w = 0; w < reps; ++w) k<NR, NW><<<148 * 8, 256>>>(in_dev, out_dev, n2);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const double bytes = (double)(NR + NW) * n2 * 16;
  printf("reads %d writes %d: %.1f us, %.0f GB/s\n", NR, NW, ms * 1e3, bytes / ms / 1e6);
  cudaFree(in_dev);
  cudaFree(out_dev);
}

int main() {
  const long n = 12830211 + 128, n2 = n / 2;
  double2 *in[8], *out[8];
  for (int a = 0; a < 8; ++a) {
    cudaMalloc(&in[a], n2 * 16);
    cudaMemset(in[a], 0, n2 * 16);
    cudaMalloc(&out[a], n2 * 16);
  }
  run<1, 1>(in, out, n2);
  run<2, 1>(in, out, n2);
  run<3, 1>(in, out, n2);
  run<4, 4>(in, out, n2);
  run<5, 4>(in, out, n2);
  run<6, 4>(in, out, n2);
  return 0;
}
