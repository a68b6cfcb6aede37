// l2_probe.cu -- development aid: does data written by one kernel survive in the B200 L2 for
// the next kernel, and does an L2 evict_first policy on a concurrent bulk stream protect it?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_probe tools/l2_probe.cu && ./l2_probe
// writer: X[i] = f(i) (S bytes), optionally also reading a bulk buffer Y (8 x S bytes, policy
// normal or evict_first);  reader: sum of X, forward or reversed sweep.  Reader time vs a cold
// read of X (L2 flushed) gives the bytes served from L2.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pol_ef() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld_ef(const double2 *p) {
  double2 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(r.x), "=d"(r.y) : "l"(p), "l"(pol_ef()));
  return r;
}
__device__ __forceinline__ double2 ld_na(const double2 *p) {
  double2 r;
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

// one thread per element of X; each also reads `ratio` elements of Y
__global__ void writer(double2 *X, long n, const double2 *Y, int ratio, int ef, int rev) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (rev) i = n - 1 - i;
  double2 acc = make_double2((double)i, 1.0);
  for (int k = 0; k < ratio; k++) {
    const double2 *p = Y + (long)k * n + i;
    double2 v = ef ? ld_ef(p) : ld_na(p);
    acc.x += v.x;
    acc.y += v.y;
  }
  X[i] = acc;
}
__global__ void reader(const double2 *X, long n, int rev, double *out) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (rev) i = n - 1 - i;
  double2 v = X[i];
  if (v.x == -1.2345) out[0] = v.y;  // never true: keeps the load
}
__global__ void flush(double2 *F, long n) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i < n) F[i] = make_double2(0.0, (double)i);
}

int main() {
  const long maxS = 400l << 20;
  double2 *X, *Y, *F;
  double *out;
  cudaMalloc(&X, maxS);
  cudaMalloc(&Y, 8 * maxS);
  cudaMalloc(&F, 512l << 20);
  cudaMalloc(&out, 8);
  cudaMemset(Y, 0, 8 * maxS);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const long nf = (512l << 20) / 16;
  auto time_read = [&](long n, int rev) {
    cudaEventRecord(a);
    reader<<<(n + 255) / 256, 256>>>(X, n, rev, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e3f;
  };
  printf("%8s %5s %3s %3s | %9s %9s %9s | %s\n", "S(MB)", "ratio", "ef", "rw", "cold_us", "fwd_us", "rev_us",
         "est. MB from L2 (rev)");
  for (long S : {32l << 20, 64l << 20, 100l << 20, 200l << 20, 400l << 20}) {
    const long n = S / 16;
    for (int ratio : {0, 4, 8}) {
      for (int ef = 0; ef < (ratio ? 2 : 1); ef++) {
        float t[3];
        for (int mode = 0; mode < 3; mode++) {  // 0 cold, 1 fwd after fwd write, 2 rev after fwd write
          float best = 1e30f;
          for (int rep = 0; rep < 5; rep++) {
            flush<<<(nf + 255) / 256, 256>>>(F, nf);
            writer<<<(n + 255) / 256, 256>>>(X, n, Y, ratio, ef, 0);
            if (mode == 0) flush<<<(nf + 255) / 256, 256>>>(F, nf);
            float us = time_read(n, mode == 2);
            best = us < best ? us : best;
          }
          t[mode] = best;
        }
        const double cold_bw = S / (t[0] * 1e-6);
        printf("%8ld %5d %3d %3s | %9.1f %9.1f %9.1f | %.0f\n", S >> 20, ratio, ef, "f", t[0], t[1], t[2],
               (t[0] - t[2]) * 1e-6 * cold_bw / 1e6);
      }
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
