// Phase timestamps of jacobi_wslice_kernel (warp 0 of every CTA, rounds 64..79) on a random n x n matrix.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2509_13224_b200/csrc tools/jw_probe.cu -o /tmp/jw_probe
long long g_ttb_launches = 0;
#include "../paper_2509_13224_b200/csrc/svd.cu"
#include <vector>
#include <random>
int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 1024;
  std::vector<double> h((size_t)n * n);
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  for (auto& x : h) x = nd(g);
  double *A, *V = nullptr;
  int *cnt, *ver, *sw;
  long long* prof;
  cudaMalloc(&A, sizeof(double) * n * n);
  cudaMalloc(&cnt, 16);
  cudaMalloc(&sw, 16);
  cudaMalloc(&ver, sizeof(int) * (n / 4 + 8) * 8);
  const int nblk = (n / 4 + 1) / 2;
  cudaMalloc(&prof, sizeof(long long) * nblk * 16 * 8);
  cudaMemset(prof, 0, sizeof(long long) * nblk * 16 * 8);
  cudaMemcpy(A, h.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
  int RW = ((((n + 7) / 8) + 15) / 16) * 16;
  size_t smem = (size_t)8 * 8 * (RW + 4) * 8;
  cudaFuncSetAttribute(jacobi_wslice_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int ms = 60;
  double tol = 4e-16 * sqrt((double)n);
  int cross = getenv("TTB_JACOBI_CROSS") ? atoi(getenv("TTB_JACOBI_CROSS")) : 1;
  void* args[] = {&n, &RW, &A, &V, &cnt, &ver, &ms, &tol, &sw, &prof, &cross};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)jacobi_wslice_kernel, dim3(nblk), dim3(WS_T), args, smem, 0);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float t; cudaEventElapsedTime(&t, e0, e1);
  int hs; cudaMemcpy(&hs, sw, 4, cudaMemcpyDeviceToHost);
  printf("launch %d (%s), n=%d, %.2f ms, sweeps %d, rounds %d, %.2f us/round\n", (int)e, cudaGetErrorString(cudaGetLastError()), n, t, hs,
         hs * (n / 4 - 1), 1e3 * t / (hs * (n / 4 - 1)));
  std::vector<long long> p((size_t)nblk * 16 * 8);
  cudaMemcpy(p.data(), prof, sizeof(long long) * p.size(), cudaMemcpyDeviceToHost);
  const char* nm[] = {"wait", "load", "gram+bar", "eigen", "apply", "fence", "release"};
  double acc[7] = {0};
  int cntr = 0;
  for (int b = 0; b < nblk; ++b)
    for (int r = 0; r < 16; ++r) {
      long long* q = &p[((size_t)b * 16 + r) * 8];
      if (!q[0] || !q[7]) continue;
      ++cntr;
      for (int k = 0; k < 7; ++k) acc[k] += (q[k + 1] ? q[k + 1] - q[k] : 0);
    }
  printf("avg over %d (CTA, round) samples, ns:", cntr);
  for (int k = 0; k < 7; ++k) printf(" %s %.0f", nm[k], acc[k] / cntr);
  printf("\n");
  // round-to-round period for CTA 0
  for (int r = 1; r < 16; ++r) printf("%lld ", p[r * 8] - p[(r - 1) * 8]);
  printf(" <- CTA0 round periods (ns)\n");
  return 0;
}
