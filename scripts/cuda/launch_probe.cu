// Launch-overhead probe: host time of <<<>>> for kernels with small / ~800 B
// parameter blocks and large dynamic shared memory, then launch->complete.
#include <chrono>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
struct Big { char b[800]; };
struct Big1k { alignas(16) char b[1100]; };
struct Big10k { alignas(16) char b[10240]; };
__global__ void __launch_bounds__(256, 1) k_gc10(const __grid_constant__ Big10k a, int* p) {
  __shared__ int st[2560];
  for (int i = threadIdx.x; i < 2560; i += blockDim.x) st[i] = reinterpret_cast<const int*>(a.b)[i];
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0 && p) *p = st[7];
}
__global__ void __launch_bounds__(256, 1) k_gc(const __grid_constant__ Big1k a, int* p) {
  extern __shared__ int s[];
  __shared__ int st[4000];
  st[threadIdx.x] = a.b[threadIdx.x % 1000];
  s[threadIdx.x] = st[threadIdx.x ^ 1];
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0 && p) *p = s[3];
}
__global__ void k_small(int* p) { if (threadIdx.x == 0 && blockIdx.x == 0 && p) *p = 1; }
__global__ void k_big(Big a, int* p) { if (threadIdx.x == 0 && blockIdx.x == 0 && p) *p = a.b[5]; }
__global__ void k_smem(Big a, int* p) {
  extern __shared__ int s[];
  s[threadIdx.x] = a.b[threadIdx.x % 800];
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0 && p) *p = s[3];
}
template <class F> void timeit(const char* name, F f, cudaStream_t st) {
  double tl = 0, tt = 0;
  const int n = 200;
  for (int i = 0; i < n + 10; ++i) {
    auto t0 = std::chrono::steady_clock::now();
    f();
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(st);
    auto t2 = std::chrono::steady_clock::now();
    if (i >= 10) {
      tl += std::chrono::duration<double, std::micro>(t1 - t0).count();
      tt += std::chrono::duration<double, std::micro>(t2 - t0).count();
    }
  }
  printf("%-28s launch %.2f us  launch+sync %.2f us\n", name, tl / n, tt / n);
}
int main() {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  int* d;
  cudaMalloc(&d, 4);
  Big b = {};
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  timeit("small, 1 block", [&] { k_small<<<1, 32, 0, st>>>(d); }, st);
  timeit("small, 148 blocks x 256", [&] { k_small<<<148, 256, 0, st>>>(d); }, st);
  timeit("800B params, 148x256", [&] { k_big<<<148, 256, 0, st>>>(b, d); }, st);
  timeit("800B + 40KB smem 148x256", [&] { k_smem<<<148, 256, 40 * 1024, st>>>(b, d); }, st);
  timeit("800B + 200KB smem attr", [&] { k_smem<<<148, 256, 4 * 1024, st>>>(b, d); }, st);
  Big1k b1 = {};
  cudaFuncSetAttribute(k_gc, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  timeit("1.1KB grid_constant 31x256", [&] { k_gc<<<31, 256, 4 * 1024, st>>>(b1, d); }, st);
  timeit("1.1KB gc + 110KB dyn smem", [&] { k_gc<<<58, 256, 110 * 1024, st>>>(b1, d); }, st);
  int* hp; cudaMallocHost(&hp, 64);
  static std::vector<char> junk(4 << 20);
  timeit("1.1KB gc + 4MB host work between", [&] {
    for (size_t i = 0; i < junk.size(); i += 64) junk[i]++;
    auto t = std::chrono::steady_clock::now();
    k_gc<<<31, 256, 4 * 1024, st>>>(b1, d);
    (void)t;
  }, st);
  static std::vector<char> small(64 << 10);
  timeit("1.1KB gc + 64KB host work", [&] {
    for (size_t i = 0; i < small.size(); i += 64) small[i]++;
    k_gc<<<31, 256, 4 * 1024, st>>>(b1, d);
  }, st);
  timeit("1.1KB gc, host-mapped out", [&] { k_gc<<<31, 256, 4 * 1024, st>>>(b1, hp); }, st);
  static Big10k b10 = {};
  timeit("10KB gc params 148x256", [&] { k_gc10<<<148, 256, 0, st>>>(b10, d); }, st);
  char* hpin; cudaMallocHost(&hpin, 16384);
  char* dbuf; cudaMalloc(&dbuf, 16384);
  timeit("10KB H2D memcpy + 1.1KB launch", [&] {
    cudaMemcpyAsync(dbuf, hpin, 9440, cudaMemcpyHostToDevice, st);
    k_gc<<<148, 256, 4 * 1024, st>>>(b1, d);
  }, st);
  timeit("1.1KB gc 148x256 alone", [&] { k_gc<<<148, 256, 4 * 1024, st>>>(b1, d); }, st);
  return 0;
}
