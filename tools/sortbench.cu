// sortbench.cu — grouping-sort microbenchmark (dev tool, not the product).
//
// Times the library's LSD radix sort (dev_radix_sort_u32, prims.cu) against
// experimental grouping kernels on a config-4 shaped key column (4 M events,
// every id in [0, 2 M) twice, the two occurrences close together).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//     -I paper_1903_06631_b200/csrc tools/sortbench.cu -o tools/sortbench \
//     -L paper_1903_06631_b200 -lmemplan_b200 -Xlinker -rpath,'$ORIGIN/../paper_1903_06631_b200'
#include <algorithm>
#include <cstdio>
#include <numeric>
#include <random>
#include <vector>

#include "common.cuh"

int dev_radix_sort_u32(mp_ctx *ctx, uint32_t *keys, uint32_t *vals, int64_t n, int bits, mp_err *err);
template <typename T>
int dev_exclusive_scan(mp_ctx *ctx, const T *in, T *out, int64_t n, T *total, mp_err *err);
extern "C" int mp_ctx_create(int device, mp_ctx **out, mp_err *err);

__global__ void k_init(const int32_t *var, int64_t n, uint32_t *keys, uint32_t *vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = (uint32_t)var[i];
    vals[i] = (uint32_t)i;
  }
}

__global__ void g_count(const int32_t *var, int64_t n, int32_t *cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[var[i]], 1);
}

__global__ void g_count4(const int4 *var4, int64_t n4, int32_t *cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    int4 v = var4[i];
    atomicAdd(&cnt[v.x], 1);
    atomicAdd(&cnt[v.y], 1);
    atomicAdd(&cnt[v.z], 1);
    atomicAdd(&cnt[v.w], 1);
  }
}

// positions from the end of each group: p = start + (count - 1 - k)
__global__ void g_scatter(const int32_t *var, int64_t n, const int32_t *start, int32_t *cnt, uint32_t *perm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = var[i];
    int32_t k = atomicSub(&cnt[v], 1);
    perm[start[v] + k - 1] = (uint32_t)i;
  }
}

__global__ void g_scatter4(const int4 *var4, int64_t n4, const int32_t *start, int32_t *cnt, uint32_t *perm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    int4 v = var4[i];
    int32_t k0 = atomicSub(&cnt[v.x], 1), k1 = atomicSub(&cnt[v.y], 1);
    int32_t k2 = atomicSub(&cnt[v.z], 1), k3 = atomicSub(&cnt[v.w], 1);
    int32_t s0 = start[v.x], s1 = start[v.y], s2 = start[v.z], s3 = start[v.w];
    perm[s0 + k0 - 1] = (uint32_t)(4 * i);
    perm[s1 + k1 - 1] = (uint32_t)(4 * i + 1);
    perm[s2 + k2 - 1] = (uint32_t)(4 * i + 2);
    perm[s3 + k3 - 1] = (uint32_t)(4 * i + 3);
  }
}

constexpr int FIX_MAX = 16;
__global__ void g_fixup(int64_t nv, const int32_t *start, int64_t n, uint32_t *perm, int32_t *nbig) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    int32_t s = start[v], e = v + 1 < nv ? start[v + 1] : (int32_t)n;
    int c = e - s;
    if (c <= 1) continue;
    if (c > FIX_MAX) { atomicAdd(nbig, 1); continue; }
    if (c == 2) {
      uint32_t a = perm[s], b = perm[s + 1];
      if (a > b) { perm[s] = b; perm[s + 1] = a; }
      continue;
    }
    uint32_t x[FIX_MAX];
    for (int i = 0; i < c; i++) x[i] = perm[s + i];
    for (int i = 1; i < c; i++) {
      uint32_t y = x[i];
      int j = i - 1;
      while (j >= 0 && x[j] > y) { x[j + 1] = x[j]; j--; }
      x[j + 1] = y;
    }
    for (int i = 0; i < c; i++) perm[s + i] = x[i];
  }
}

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

int main(int argc, char **argv) {
  const int64_t nvars = 2000000, n = 2 * nvars;
  std::mt19937_64 rng(1);
  std::vector<int32_t> ids(nvars);
  std::iota(ids.begin(), ids.end(), 0);
  std::shuffle(ids.begin(), ids.end(), rng);
  // malloc of ids[i] at slot 2i, free at 2(i + len) + 1: stable order by slot
  std::vector<std::pair<int64_t, int32_t>> ev;
  ev.reserve(n);
  for (int64_t i = 0; i < nvars; i++) {
    int64_t len = 1 + (int64_t)(rng() % 63);
    ev.push_back({2 * i, ids[i]});
    ev.push_back({2 * std::min(i + len, nvars - 1) + 1, ids[i]});
  }
  std::stable_sort(ev.begin(), ev.end(), [](auto &a, auto &b) { return a.first < b.first; });
  std::vector<int32_t> var(n);
  for (int64_t i = 0; i < n; i++) var[i] = ev[i].second;

  mp_ctx *ctx;
  mp_err err{};
  if (mp_ctx_create(0, &ctx, &err)) { printf("ctx failed\n"); return 1; }
  cudaStream_t st = ctx->stream;
  int32_t *d_var, *cnt, *start, *nbig;
  uint32_t *keys, *vals, *perm;
  CK(cudaMalloc(&d_var, n * 4));
  CK(cudaMalloc(&keys, n * 4));
  CK(cudaMalloc(&vals, n * 4));
  CK(cudaMalloc(&perm, n * 4));
  CK(cudaMalloc(&cnt, (nvars + 1) * 4));
  CK(cudaMalloc(&start, (nvars + 1) * 4));
  CK(cudaMalloc(&nbig, 4));
  CK(cudaMemcpy(d_var, var.data(), n * 4, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = ctx->num_sms;
  auto timeit = [&](const char *name, auto fn) {
    for (int w = 0; w < 3; w++) fn();
    cudaStreamSynchronize(st);
    float best = 1e9, tot = 0;
    for (int r = 0; r < 20; r++) {
      cudaEventRecord(e0, st);
      fn();
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = std::min(best, ms);
      tot += ms;
    }
    printf("%-40s best %8.1f us  mean %8.1f us\n", name, best * 1e3, tot / 20 * 1e3);
  };
  // reference: stable sort (key, index) on the host
  std::vector<uint32_t> want(n);
  {
    std::vector<int64_t> cntv(nvars + 1, 0);
    for (int64_t i = 0; i < n; i++) cntv[var[i] + 1]++;
    for (int64_t v = 0; v < nvars; v++) cntv[v + 1] += cntv[v];
    for (int64_t i = 0; i < n; i++) want[cntv[var[i]]++] = (uint32_t)i;
  }
  auto check = [&](const uint32_t *d, const char *name) {
    std::vector<uint32_t> got(n);
    cudaMemcpy(got.data(), d, n * 4, cudaMemcpyDeviceToHost);
    printf("  %s %s\n", name, got == want ? "OK" : "MISMATCH");
  };
  int bits = 21;
  timeit("radix (init + 3 x 8-bit passes)", [&] {
    k_init<<<grid_for(n, 256), 256, 0, st>>>(d_var, n, keys, vals);
    dev_radix_sort_u32(ctx, keys, vals, n, bits, &err);
  });
  check(vals, "radix");
  auto group = [&](bool vec) {
    cudaMemsetAsync(cnt, 0, (nvars + 1) * 4, st);
    cudaMemsetAsync(nbig, 0, 4, st);
    if (vec) g_count4<<<grid_for(n / 4, 256, sms * 16), 256, 0, st>>>((const int4 *)d_var, n / 4, cnt);
    else g_count<<<grid_for(n, 256, sms * 16), 256, 0, st>>>(d_var, n, cnt);
    dev_exclusive_scan<int32_t>(ctx, cnt, start, nvars, nullptr, &err);
    if (vec) g_scatter4<<<grid_for(n / 4, 256, sms * 16), 256, 0, st>>>((const int4 *)d_var, n / 4, start, cnt, perm);
    else g_scatter<<<grid_for(n, 256, sms * 16), 256, 0, st>>>(d_var, n, start, cnt, perm);
    g_fixup<<<grid_for(nvars, 256), 256, 0, st>>>(nvars, start, n, perm, nbig);
  };
  timeit("count+scan+scatter+fixup", [&] { group(false); });
  check(perm, "group");
  timeit("count+scan+scatter+fixup (int4)", [&] { group(true); });
  check(perm, "group4");
  {
    // placement-order shape: 1 M keys, 26-bit sizes, values 0..n-1
    const int64_t m = 1000000;
    std::vector<uint32_t> hk(m);
    for (auto &x : hk) x = (uint32_t)(rng() % ((1u << 26) - 512));
    std::vector<uint32_t> wantv(m);
    std::iota(wantv.begin(), wantv.end(), 0u);
    std::stable_sort(wantv.begin(), wantv.end(), [&](uint32_t a, uint32_t b) { return hk[a] < hk[b]; });
    uint32_t *k2, *v2, *k0;
    CK(cudaMalloc(&k2, m * 4));
    CK(cudaMalloc(&v2, m * 4));
    CK(cudaMalloc(&k0, m * 4));
    CK(cudaMemcpy(k0, hk.data(), m * 4, cudaMemcpyHostToDevice));
    timeit("order: 1M x 26-bit (copy + sort)", [&] {
      cudaMemcpyAsync(k2, k0, m * 4, cudaMemcpyDeviceToDevice, st);
      k_init<<<grid_for(m, 256), 256, 0, st>>>((const int32_t *)k0, m, k2, v2);
      dev_radix_sort_u32(ctx, k2, v2, m, 26, &err);
    });
    std::vector<uint32_t> got(m);
    cudaMemcpy(got.data(), v2, m * 4, cudaMemcpyDeviceToHost);
    printf("  order %s\n", got == wantv ? "OK" : "MISMATCH");
  }
  timeit("  count only", [&] {
    cudaMemsetAsync(cnt, 0, (nvars + 1) * 4, st);
    g_count<<<grid_for(n, 256, sms * 16), 256, 0, st>>>(d_var, n, cnt);
  });
  timeit("  scan only", [&] { dev_exclusive_scan<int32_t>(ctx, cnt, start, nvars, nullptr, &err); });
  return 0;
}
