// FMA-pipe microbenchmark for B200 (sm_100a): FP64 / FP32 FMA throughput and
// dependent-chain latency. Used to derive the ALU roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T, int CH>
__global__ void thr(T* out, int iters, T a, T b) {
  T x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = (T)(threadIdx.x + c) * (T)1e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = x[c] * a + b;
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == (T)12345.678) out[0] = s;
}
// the fit loop's form: every operand a distinct register (coefficients held
// in registers per chain, as fma(A, f, c) in run_propagator)
template <typename T, int CH>
__global__ void thr_reg(T* out, const T* coef, int iters) {
  T x[CH], a[CH], b[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    x[c] = (T)(threadIdx.x + c) * (T)1e-3;
    a[c] = coef[c];
    b[c] = coef[CH + c];
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a[c], b[c]);
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == (T)12345.678) out[0] = s;
}
template <typename T, int CH>
void run_thr_reg(const char* name, int blocks, int threads, int iters) {
  T* d; cudaMalloc(&d, 64);
  T hc[2 * CH];
  for (int c = 0; c < 2 * CH; ++c) hc[c] = c < CH ? (T)(0.999999 - 1e-7 * c) : (T)(1e-7 * (c + 1));
  T* dc; cudaMalloc(&dc, sizeof(hc)); cudaMemcpy(dc, hc, sizeof(hc), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  thr_reg<T, CH><<<blocks, threads>>>(d, dc, iters);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) thr_reg<T, CH><<<blocks, threads>>>(d, dc, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fma = 5.0 * blocks * threads * (double)iters * CH;
  printf("%s 3-reg blocks=%d threads=%d chains=%d: %.3f TFMA/s = %.2f TFLOP/s (%.3f ms)\n", name, blocks,
         threads, CH, fma / (ms * 1e-3) / 1e12, 2 * fma / (ms * 1e-3) / 1e12, ms);
  cudaFree(d); cudaFree(dc);
}
// FFMA2 (sm_100: two fp32 FMAs per instruction), the fit loop's packed form:
// x2 = fma2(A2, (s, s), x2) with the multiplier broadcast from one register
template <int CH>
__global__ void thr_ffma2(float2* out, const float* coef, int iters) {
  float2 x[CH], a[CH];
  float s[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    x[c] = make_float2((threadIdx.x + c) * 1e-3f, (threadIdx.x + c) * 2e-3f);
    a[c] = make_float2(coef[c], coef[CH + c]);
    s[c] = coef[2 * CH + c];
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __ffma2_rn(a[c], make_float2(s[c], s[c]), x[c]);
  }
  float t = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) t += x[c].x + x[c].y;
  if (t == 12345.678f) out[0] = x[0];
}
template <int CH>
void run_ffma2(int blocks, int threads, int iters) {
  float2* d; cudaMalloc(&d, 64);
  float hc[3 * CH];
  for (int c = 0; c < 3 * CH; ++c) hc[c] = c < 2 * CH ? 0.999999f - 1e-7f * c : 1e-7f * (c + 1);
  float* dc; cudaMalloc(&dc, sizeof(hc)); cudaMemcpy(dc, hc, sizeof(hc), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  thr_ffma2<CH><<<blocks, threads>>>(d, dc, iters);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) thr_ffma2<CH><<<blocks, threads>>>(d, dc, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fma = 5.0 * blocks * threads * (double)iters * CH * 2;
  printf("FFMA2 (broadcast, 3-reg) blocks=%d threads=%d chains=%d: %.3f TFMA/s = %.2f TFLOP/s (%.3f ms)\n",
         blocks, threads, CH, fma / (ms * 1e-3) / 1e12, 2 * fma / (ms * 1e-3) / 1e12, ms);
  cudaFree(d); cudaFree(dc);
}
template <typename T>
__global__ void lat(T* out, long long* cyc, int iters, T a, T b) {
  T x = (T)threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = x * a + b; x = x * a + b; x = x * a + b; x = x * a + b; }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; }
  if (x == (T)12345.678) out[0] = x;
}
template <typename T, int CH>
void run_thr(const char* name, int blocks, int threads, int iters) {
  T* d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  thr<T, CH><<<blocks, threads>>>(d, iters, (T)0.999999, (T)1e-7);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) thr<T, CH><<<blocks, threads>>>(d, iters, (T)0.999999, (T)1e-7);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fma = 5.0 * blocks * threads * (double)iters * CH;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%s blocks=%d threads=%d chains=%d: %.3f TFMA/s = %.2f TFLOP/s (%.3f ms)\n", name, blocks, threads, CH,
         fma / (ms * 1e-3) / 1e12, 2 * fma / (ms * 1e-3) / 1e12, ms);
  cudaFree(d);
}
template <typename T>
void run_lat(const char* name) {
  T* d; long long* c; cudaMalloc(&d, 64); cudaMalloc(&c, 8);
  int iters = 4096;
  lat<T><<<1, 32>>>(d, c, iters, (T)0.999999, (T)1e-7);
  lat<T><<<1, 32>>>(d, c, iters, (T)0.999999, (T)1e-7);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%s dependent latency: %.2f cycles\n", name, (double)h / (4.0 * iters));
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("%s SMs=%d clock=%d kHz regs/SM=%d smem/SM=%zu\n", p.name, p.multiProcessorCount, p.clockRate,
         p.regsPerMultiprocessor, p.sharedMemPerMultiprocessor);
  int sm = p.multiProcessorCount;
  run_lat<double>("DFMA");
  run_lat<float>("FFMA");
  for (int w : {4, 8, 16, 32}) run_thr<double, 8>("DFMA", sm * (w / 4), 128, 20000);
  run_thr<double, 4>("DFMA", sm * 4, 128, 20000);
  run_thr<double, 2>("DFMA", sm * 8, 128, 20000);
  for (int w : {4, 8, 16, 32}) run_thr<float, 8>("FFMA", sm * (w / 4), 128, 40000);
  for (int w : {8, 16, 32}) run_thr_reg<float, 8>("FFMA", sm * (w / 4), 128, 40000);
  for (int w : {8, 16, 32}) run_thr_reg<double, 8>("DFMA", sm * (w / 4), 128, 20000);
  for (int w : {8, 16, 32}) run_ffma2<8>(sm * (w / 4), 128, 40000);
  return 0;
}
