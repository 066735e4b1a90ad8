// Checks the m8n8k4 f64 fragment layout assumed by ax_mma.cu on the device:
// A[g][q] (lane 4g+q), B[q][g], C[g][2q+i].  Prints PASS/FAIL.
#include <cstdio>
#include <cmath>
__global__ void k(double* out) {
  const int l = threadIdx.x, g = l >> 2, q = l & 3;
  const double a = 1.0 + g * 4 + q;        // A[g][q]
  const double b = 0.5 + q * 8 + g * 0.25; // B[q][g]
  double d0, d1;
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
      : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(0.0), "d"(0.0));
  out[g * 8 + 2 * q] = d0;
  out[g * 8 + 2 * q + 1] = d1;
}
int main() {
  double* d; cudaMalloc(&d, 64 * 8);
  k<<<1, 32>>>(d);
  double h[64]; cudaMemcpy(h, d, 512, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < 8; ++r) for (int c = 0; c < 8; ++c) {
    double s = 0; for (int kk = 0; kk < 4; ++kk) s += (1.0 + r * 4 + kk) * (0.5 + kk * 8 + c * 0.25);
    if (fabs(s - h[r * 8 + c]) > 1e-9) { if (bad < 5) printf("C[%d][%d] = %g want %g\n", r, c, h[r * 8 + c], s); ++bad; }
  }
  printf(bad ? "FAIL %d\n" : "PASS\n", bad);
  return 0;
}
