// Orthogonality (c^2 + s^2 - 1: max and mean, i.e. bias) of jrot_fast vs jrot over random 2x2 Grams.
long long g_ttb_launches = 0;
#include "../paper_2509_13224_b200/csrc/svd.cu"
#include <curand_kernel.h>
__global__ void k(double* out, int fast) {
  curandStatePhilox4_32_10_t st;
  curand_init(1234, blockIdx.x * blockDim.x + threadIdx.x, 0, &st);
  double mx = 0, sum = 0;
  for (int i = 0; i < 1000; ++i) {
    double a = exp(8 * curand_normal_double(&st)), b = exp(8 * curand_normal_double(&st));
    double g = curand_normal_double(&st) * sqrt(a * b) * 0.5;
    double c, s;
    if (fast) jrot_fast(a, b, g, 1e-32, c, s); else jrot(a, b, g, 1e-32, true, c, s);
    double e = fma(c, c, fma(s, s, -1.0));
    mx = fmax(mx, fabs(e)); sum += e;
  }
  atomicAdd(out, sum);
  unsigned long long* m = (unsigned long long*)(out + 1);
  atomicMax(m, __double_as_longlong(mx));
}
int main() {
  for (int fast = 0; fast < 2; ++fast) {
    double* o; cudaMalloc(&o, 16); cudaMemset(o, 0, 16);
    k<<<256, 256>>>(o, fast);
    double h[2]; cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
    printf("%s: mean(c^2+s^2-1) = %.3e, max |.| = %.3e\n", fast ? "jrot_fast" : "jrot", h[0] / (256.0 * 256 * 1000), h[1]);
  }
}
