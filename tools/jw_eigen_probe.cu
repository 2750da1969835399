// Cycle count of the warp-level 8 x 8 Jacobi sweep (jw_eigen8) and of its rotation (jrot_fast).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/jw_eigen_probe.cu -o tools/jw_eigen_probe.bin
long long g_ttb_launches = 0;
#include "../paper_2509_13224_b200/csrc/svd.cu"
__global__ void probe(const double* G0, double* out, long long* cyc, int reps, int reg) {
  __shared__ double G[64], J[64];
  const int lane = threadIdx.x;
  long long t0 = 0, acc = 0;
  for (int r = 0; r < reps; ++r) {
    for (int e = lane; e < 64; e += 32) { G[e] = G0[e]; J[e] = ((e >> 3) == (e & 7)) ? 1.0 : 0.0; }
    __syncwarp();
    t0 = clock64();
    bool nd = jw_eigen8(G, J, 1e-14, lane);
    __syncwarp();
    acc += clock64() - t0;
    if (!nd) out[0] += 1.0;
  }
  // rotation chain alone
  double a = G0[0], b = G0[9], g = G0[1], c = 0, s = 0;
  long long t1 = clock64();
  for (int r = 0; r < 100; ++r) { jrot_fast(a, b, g, 1e-30, c, s); a += c * 1e-30; g += s * 1e-30; }
  long long t2 = clock64();
  for (int e = lane; e < 64; e += 32) out[1 + e] = J[e];
  if (lane == 0) { cyc[0] = acc / reps; cyc[1] = (t2 - t1) / 100; out[65] = a + g; }
}
int main() {
  double h[64];
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 8; ++j) h[i * 8 + j] = (i == j ? 10.0 + i : 0.1 * (i + j + 1));
  double *G0, *out; long long* cyc;
  cudaMalloc(&G0, 512); cudaMalloc(&out, 66 * 8); cudaMalloc(&cyc, 16);
  cudaMemcpy(G0, h, 512, cudaMemcpyHostToDevice); cudaMemset(out, 0, 66 * 8);
  for (int reg = 0; reg < 1; ++reg) {
    probe<<<1, 32>>>(G0, out, cyc, 100, reg);
    long long hc[2]; cudaMemcpy(hc, cyc, 16, cudaMemcpyDeviceToHost);
    double hJ[66]; cudaMemcpy(hJ, out, 66 * 8, cudaMemcpyDeviceToHost);
    // off-diagonal mass of J^T G J
    double M[64];
    for (int a = 0; a < 8; ++a) for (int b = 0; b < 8; ++b) { double t = 0; for (int x = 0; x < 8; ++x) for (int y = 0; y < 8; ++y) t += hJ[1 + x * 8 + a] * h[x * 8 + y] * hJ[1 + y * 8 + b]; M[a * 8 + b] = t; }
    double off = 0, orth = 0;
    for (int a = 0; a < 8; ++a) for (int b = 0; b < 8; ++b) { if (a != b) off += M[a * 8 + b] * M[a * 8 + b];
      double t = 0; for (int x = 0; x < 8; ++x) t += hJ[1 + x * 8 + a] * hJ[1 + x * 8 + b]; orth = fmax(orth, fabs(t - (a == b))); }
    printf("%s: %lld cycles per call (7 rounds), jrot_fast chain: %lld cycles, off-diag after one sweep %.3e, J orth %.1e\n",
           reg ? "jw_eigen8_reg" : "jw_eigen8", hc[0], hc[1], sqrt(off), orth);
  }
}
