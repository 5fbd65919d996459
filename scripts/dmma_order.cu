// Does mma.sync.m8n8k4 f64 on sm_100a compute d = fma(a3,b3,fma(a2,b2,fma(a1,b1,fma(a0,b0,c))))?
// Compares every element of D against the sequential fma chain (k order) and
// against the unfused sum, over random tiles.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

__global__ void dmma(const double* A, const double* B, const double* C, double* D) {
  const int lane = threadIdx.x;
  const double a = A[(lane >> 2) * 4 + (lane & 3)];        // A 8x4 row-major: row lane/4, col lane%4
  const double b = B[(lane & 3) * 8 + (lane >> 2)];        // B 4x8: row lane%4, col lane/4
  double c0 = C[(lane >> 2) * 8 + (lane & 3) * 2], c1 = C[(lane >> 2) * 8 + (lane & 3) * 2 + 1];
  double d0, d1;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
  D[(lane >> 2) * 8 + (lane & 3) * 2] = d0;
  D[(lane >> 2) * 8 + (lane & 3) * 2 + 1] = d1;
}

int main() {
  double *A, *B, *C, *D;
  cudaMallocManaged(&A, 32 * 8); cudaMallocManaged(&B, 32 * 8); cudaMallocManaged(&C, 64 * 8); cudaMallocManaged(&D, 64 * 8);
  srand(1);
  long same_fma = 0, same_plain = 0, total = 0;
  for (int trial = 0; trial < 2000; ++trial) {
    for (int i = 0; i < 32; ++i) { A[i] = (rand() / (double)RAND_MAX - 0.5) * pow(10.0, rand() % 6 - 3); B[i] = (rand() / (double)RAND_MAX - 0.5) * pow(10.0, rand() % 6 - 3); }
    for (int i = 0; i < 64; ++i) C[i] = (rand() / (double)RAND_MAX - 0.5) * pow(10.0, rand() % 6 - 3);
    dmma<<<1, 32>>>(A, B, C, D);
    cudaDeviceSynchronize();
    for (int r = 0; r < 8; ++r)
      for (int c = 0; c < 8; ++c) {
        double s = C[r * 8 + c], p = C[r * 8 + c];
        for (int k = 0; k < 4; ++k) { s = fma(A[r * 4 + k], B[k * 8 + c], s); p = p + A[r * 4 + k] * B[k * 8 + c]; }
        same_fma += (s == D[r * 8 + c]);
        same_plain += (p == D[r * 8 + c]);
        ++total;
      }
  }
  printf("{\"elements\": %ld, \"equal_sequential_fma\": %ld, \"equal_unfused\": %ld}\n", total, same_fma, same_plain);
  return 0;
}
