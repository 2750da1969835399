// Classical full-grid IGA system on the device: the independent equivalence anchor of the TT pipeline
// (reference driver.py:561-703, full_grid_reference: sparse element-by-element assembly with the same
// quadrature, Dirichlet elimination, direct/CG solve). Used only by driver.full_grid_reference.
//
// Storage: the stiffness of a tensor-product B-spline space couples dof i only with dofs j whose
// per-direction indices differ by at most p_d, so K is kept as a stencil array K[i][s] with
// s = ((o0 (2p1+1) + o1) (2p2+1) + o2), o_d = j_d - i_d + p_d (n_dofs x prod(2p_d+1) FP64) -- a
// banded layout, converted to CSR on the host only for the API's return value.
#include "common.cuh"

namespace {

struct FgArgs {
  int ne[3], g[3], p[3], n[3];
  const int* starts[3];   // first active basis index per quadrature point
  const double* V[3];     // (nq, p+1) values
  const double* D[3];     // (nq, p+1) derivatives
  const double* Rw;       // (nq0 nq1 nq2, 9): w0 w1 w2 R_ij at every quadrature point
  const double* Fw;       // (nq0 nq1 nq2): w0 w1 w2 f(x) det J
};

constexpr int FG_T = 256;
constexpr int FG_MAXQ = 512;     // quadrature points per element held in shared memory (g0 g1 g2)
constexpr int FG_MAXT = 16;      // points per direction
constexpr int FG_MAXP = 8;       // basis functions per direction (p + 1)

// One CTA per element: local stiffness entries (a, b) over the element's g0 g1 g2 points, scattered into
// the stencil rows with atomics (elements sharing a dof add into the same entries); local load likewise.
__global__ void __launch_bounds__(FG_T) fullgrid_elem_kernel(FgArgs A, double* __restrict__ K, double* __restrict__ f) {
  __shared__ double Rs[FG_MAXQ * 9];
  __shared__ double Fs[FG_MAXQ];
  __shared__ double Vs[3][FG_MAXT][FG_MAXP], Ds[3][FG_MAXT][FG_MAXP];
  const int e = blockIdx.x;
  const int e2 = e % A.ne[2], e1 = (e / A.ne[2]) % A.ne[1], e0 = e / (A.ne[2] * A.ne[1]);
  const int ee[3] = {e0, e1, e2};
  const int g0 = A.g[0], g1 = A.g[1], g2 = A.g[2];
  const int nq1 = A.ne[1] * g1, nq2 = A.ne[2] * g2;
  const int nqe = g0 * g1 * g2;
  for (int t = threadIdx.x; t < nqe; t += blockDim.x) {
    const int t2 = t % g2, t1 = (t / g2) % g1, t0 = t / (g2 * g1);
    const long long q = ((long long)(e0 * g0 + t0) * nq1 + (e1 * g1 + t1)) * nq2 + (e2 * g2 + t2);
#pragma unroll
    for (int c = 0; c < 9; ++c) Rs[t * 9 + c] = A.Rw[q * 9 + c];
    Fs[t] = A.Fw[q];
  }
  for (int d = 0; d < 3; ++d)
    for (int it = threadIdx.x; it < A.g[d] * (A.p[d] + 1); it += blockDim.x) {
      const int t = it / (A.p[d] + 1), a = it % (A.p[d] + 1);
      const long long q = (long long)ee[d] * A.g[d] + t;
      Vs[d][t][a] = A.V[d][q * (A.p[d] + 1) + a];
      Ds[d][t][a] = A.D[d][q * (A.p[d] + 1) + a];
    }
  __syncthreads();
  const int m0 = A.p[0] + 1, m1 = A.p[1] + 1, m2 = A.p[2] + 1;
  const int nloc = m0 * m1 * m2;
  int s[3];
  for (int d = 0; d < 3; ++d) s[d] = A.starts[d][(long long)ee[d] * A.g[d]];
  const int w1 = 2 * A.p[1] + 1, w2 = 2 * A.p[2] + 1;
  const int S = (2 * A.p[0] + 1) * w1 * w2;
  for (int pr = threadIdx.x; pr < nloc * nloc; pr += blockDim.x) {
    const int a = pr / nloc, b = pr % nloc;
    const int a2 = a % m2, a1 = (a / m2) % m1, a0 = a / (m2 * m1);
    const int b2 = b % m2, b1 = (b / m2) % m1, b0 = b / (m2 * m1);
    double acc = 0.0;
    int t = 0;
    for (int t0 = 0; t0 < g0; ++t0) {
      const double va0 = Vs[0][t0][a0], da0 = Ds[0][t0][a0], vb0 = Vs[0][t0][b0], db0 = Ds[0][t0][b0];
      for (int t1 = 0; t1 < g1; ++t1) {
        const double va1 = Vs[1][t1][a1], da1 = Ds[1][t1][a1], vb1 = Vs[1][t1][b1], db1 = Ds[1][t1][b1];
        for (int t2 = 0; t2 < g2; ++t2, ++t) {
          const double va2 = Vs[2][t2][a2], da2 = Ds[2][t2][a2], vb2 = Vs[2][t2][b2], db2 = Ds[2][t2][b2];
          const double ga[3] = {da0 * va1 * va2, va0 * da1 * va2, va0 * va1 * da2};
          const double gb[3] = {db0 * vb1 * vb2, vb0 * db1 * vb2, vb0 * vb1 * db2};
          const double* R = Rs + t * 9;
#pragma unroll
          for (int i = 0; i < 3; ++i) acc += ga[i] * (R[3 * i] * gb[0] + R[3 * i + 1] * gb[1] + R[3 * i + 2] * gb[2]);
        }
      }
    }
    const long long row = ((long long)(s[0] + a0) * A.n[1] + (s[1] + a1)) * A.n[2] + (s[2] + a2);
    const int slot = ((b0 - a0 + A.p[0]) * w1 + (b1 - a1 + A.p[1])) * w2 + (b2 - a2 + A.p[2]);
    atomicAdd(K + row * S + slot, acc);
  }
  for (int a = threadIdx.x; a < nloc; a += blockDim.x) {
    const int a2 = a % m2, a1 = (a / m2) % m1, a0 = a / (m2 * m1);
    double acc = 0.0;
    int t = 0;
    for (int t0 = 0; t0 < g0; ++t0)
      for (int t1 = 0; t1 < g1; ++t1)
        for (int t2 = 0; t2 < g2; ++t2, ++t) acc += Vs[0][t0][a0] * Vs[1][t1][a1] * Vs[2][t2][a2] * Fs[t];
    const long long row = ((long long)(s[0] + a0) * A.n[1] + (s[1] + a1)) * A.n[2] + (s[2] + a2);
    atomicAdd(f + row, acc);
  }
}

// y = M K M x (M = diag(mask), mask == nullptr: identity) on the stencil storage; one thread per row.
__global__ void stencil_spmv_kernel(int n0, int n1, int n2, int p0, int p1, int p2, const double* __restrict__ K,
                                    const double* __restrict__ x, const unsigned char* __restrict__ mask,
                                    double* __restrict__ y) {
  const long long N = (long long)n0 * n1 * n2;
  const int w1 = 2 * p1 + 1, w2 = 2 * p2 + 1;
  const int S = (2 * p0 + 1) * w1 * w2;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    if (mask && !mask[i]) { y[i] = 0.0; continue; }
    const int i2 = (int)(i % n2), i1 = (int)((i / n2) % n1), i0 = (int)(i / ((long long)n2 * n1));
    const double* Ki = K + i * S;
    double acc = 0.0;
    for (int o0 = -p0; o0 <= p0; ++o0) {
      const int j0 = i0 + o0;
      if (j0 < 0 || j0 >= n0) continue;
      for (int o1 = -p1; o1 <= p1; ++o1) {
        const int j1 = i1 + o1;
        if (j1 < 0 || j1 >= n1) continue;
        const double* Kr = Ki + ((o0 + p0) * w1 + (o1 + p1)) * w2 + p2;
        const long long jb = ((long long)j0 * n1 + j1) * n2;
        for (int o2 = -p2; o2 <= p2; ++o2) {
          const int j2 = i2 + o2;
          if (j2 < 0 || j2 >= n2) continue;
          const long long j = jb + j2;
          if (mask && !mask[j]) continue;
          acc += Kr[o2] * x[j];
        }
      }
    }
    y[i] = acc;
  }
}

}  // namespace

TTB_API int ttb_fullgrid_assemble(void* stream, const int* ne, const int* g, const int* p, const int* n,
                                  const int* s0, const int* s1, const int* s2, const double* V0, const double* V1,
                                  const double* V2, const double* D0, const double* D1, const double* D2,
                                  const double* Rw, const double* Fw, double* K, double* f) {
  FgArgs A;
  for (int d = 0; d < 3; ++d) {
    A.ne[d] = ne[d]; A.g[d] = g[d]; A.p[d] = p[d]; A.n[d] = n[d];
    if (ne[d] < 1 || g[d] < 1 || g[d] > FG_MAXT || p[d] < 0 || p[d] + 1 > FG_MAXP) return TTB_EARG;
  }
  if ((long long)g[0] * g[1] * g[2] > FG_MAXQ) return TTB_EARG;
  A.starts[0] = s0; A.starts[1] = s1; A.starts[2] = s2;
  A.V[0] = V0; A.V[1] = V1; A.V[2] = V2;
  A.D[0] = D0; A.D[1] = D1; A.D[2] = D2;
  A.Rw = Rw;
  A.Fw = Fw;
  const long long nel = (long long)ne[0] * ne[1] * ne[2];
  if (nel > 0x7fffffffLL) return TTB_EARG;
  fullgrid_elem_kernel<<<(unsigned)nel, FG_T, 0, as_stream(stream)>>>(A, K, f); ttb_count();
  return ttb_last_error();
}

TTB_API int ttb_stencil_spmv(void* stream, int n0, int n1, int n2, int p0, int p1, int p2, const double* K,
                             const double* x, const unsigned char* mask, double* y) {
  const long long N = (long long)n0 * n1 * n2;
  if (N <= 0) return TTB_OK;
  const long long blocks = (N + 255) / 256 < ttb_num_sms() * 16 ? (N + 255) / 256 : ttb_num_sms() * 16;
  stencil_spmv_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(n0, n1, n2, p0, p1, p2, K, x, mask, y); ttb_count();
  return ttb_last_error();
}
