// lb_abi: the multi-process kernels in a loopback world, driven through the C ABI
// alone (include/rp.h) -- no Python, no PyTorch allocator, no pageable copies.
// W ranks = W host threads in this process, one non-blocking stream each, all on
// device 0 (rp_comm_set_loopback). A seeded random sequence of all_reduce (sum /
// max, user and in-place buffers, one-shot and two-shot sizes), all_gather and
// broadcast runs back to back; every result is compared bit for bit with the
// rank-ordered fold computed on the host. Meant as the first, minimal contact with a
// GPU under compute-sanitizer (tools/runs/r02_safety.sh), and as a C++ example of
// the C-ABI seam (INTEGRATION.md seam 3).
//
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/lb_abi.cu \
//        -Lpaper_1902_00465_b200 -lrp -Xlinker -rpath,'$ORIGIN/../paper_1902_00465_b200' -o tools/lb_abi
//   tools/lb_abi W N_OPS SEED
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include <condition_variable>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../include/rp.h"

namespace {

struct Barrier {
  std::mutex m;
  std::condition_variable cv;
  int n, waiting = 0, gen = 0;
  explicit Barrier(int n_) : n(n_) {}
  void wait() {
    std::unique_lock<std::mutex> l(m);
    const int g = gen;
    if (++waiting == n) {
      waiting = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(l, [&] { return gen != g; });
    }
  }
};

struct Op {
  int kind;  // 0 all_reduce sum, 1 all_reduce max (in place), 2 all_gather, 3 broadcast
  size_t count;
  int root;
};

// deterministic input of rank r for op i (same on every thread)
float value(uint32_t seed, int i, int r, size_t k) {
  uint32_t h = seed * 2654435761u ^ (uint32_t)i * 40503u ^ (uint32_t)r * 2246822519u ^ (uint32_t)k * 3266489917u;
  h ^= h >> 15;
  h *= 2246822519u;
  h ^= h >> 13;
  return ((float)(h & 0xFFFFFF) / 16777216.0f - 0.5f) * 8.0f;
}

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      fprintf(stderr, "rank %d: %s: %s\n", rank, #x, cudaGetErrorString(e_));             \
      _exit(2); /* peers would wait at the host barrier forever */                         \
    }                                                                                      \
  } while (0)
#define RP(x)                                                                              \
  do {                                                                                     \
    int rc_ = (x);                                                                         \
    if (rc_ != RP_OK) {                                                                    \
      fprintf(stderr, "rank %d: %s -> %d: %s\n", rank, #x, rc_, rp_last_error());         \
      _exit(2);                                                                            \
    }                                                                                      \
  } while (0)

int rank_main(int rank, int W, const std::vector<Op>& ops, uint32_t seed, Barrier& bar,
              std::vector<std::string>& blobs, long* bad_out) {
  CK(cudaSetDevice(0));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  size_t maxc = 1;
  for (const Op& o : ops) maxc = std::max(maxc, o.count);
  // every allocation before the first collective: nothing may wait on the device
  // while a peer's kernel waits for this rank
  float *x = nullptr, *y = nullptr, *hx = nullptr, *hy = nullptr;
  CK(cudaMalloc(&x, maxc * 4));
  CK(cudaMalloc(&y, maxc * W * 4));
  CK(cudaMallocHost(&hx, maxc * 4));
  CK(cudaMallocHost(&hy, maxc * W * 4));
  rp_comm_t c = nullptr;
  RP(rp_comm_create(rank, W, 0, (size_t)64 << 20, &c));
  RP(rp_comm_set_loopback(c, 1));
  RP(rp_comm_set_timeout(c, 10ull * 1000 * 1000 * 1000));
  std::string blob(rp_comm_export_size(), '\0');
  size_t n = blob.size();
  RP(rp_comm_export(c, &blob[0], &n));
  blobs[rank] = blob;
  bar.wait();
  std::string all;
  for (const std::string& b : blobs) all += b;
  bar.wait();
  RP(rp_comm_import(c, all.data(), all.size()));
  long bad = 0;
  std::vector<float> want(maxc * W);
  for (size_t i = 0; i < ops.size(); ++i) {
    const Op& o = ops[i];
    for (size_t k = 0; k < o.count; ++k) hx[k] = value(seed, (int)i, rank, k);
    CK(cudaMemcpyAsync(x, hx, o.count * 4, cudaMemcpyHostToDevice, s));
    size_t outn = o.count;
    if (o.kind == 0) {
      RP(rp_all_reduce(c, x, y, o.count, RP_F32, RP_F32, RP_F32, RP_SUM, RP_ALGO_AUTO, s));
      for (size_t k = 0; k < o.count; ++k) {
        float acc = value(seed, (int)i, 0, k);
        for (int p = 1; p < W; ++p) acc = acc + value(seed, (int)i, p, k);  // ascending rank
        want[k] = acc;
      }
    } else if (o.kind == 1) {
      RP(rp_all_reduce(c, x, x, o.count, RP_F32, RP_F32, RP_F32, RP_MAX, RP_ALGO_AUTO, s));
      CK(cudaMemcpyAsync(y, x, o.count * 4, cudaMemcpyDeviceToDevice, s));
      for (size_t k = 0; k < o.count; ++k) {
        float acc = value(seed, (int)i, 0, k);
        for (int p = 1; p < W; ++p) {
          const float v = value(seed, (int)i, p, k);
          acc = (acc > v || acc != acc) ? acc : v;  // np.maximum select
        }
        want[k] = acc;
      }
    } else if (o.kind == 2) {
      RP(rp_all_gather(c, x, y, o.count * 4, s));
      outn = o.count * W;
      for (int p = 0; p < W; ++p)
        for (size_t k = 0; k < o.count; ++k) want[p * o.count + k] = value(seed, (int)i, p, k);
    } else {
      RP(rp_broadcast(c, x, y, o.count * 4, o.root, RP_ALGO_AUTO, s));
      for (size_t k = 0; k < o.count; ++k) want[k] = value(seed, (int)i, o.root, k);
    }
    CK(cudaMemcpyAsync(hy, y, outn * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    long b = 0;
    for (size_t k = 0; k < outn; ++k) b += memcmp(&hy[k], &want[k], 4) != 0;
    if (b) fprintf(stderr, "rank %d op %zu (kind %d, %zu elements): %ld mismatches\n", rank, i, o.kind, o.count, b);
    bad += b;
  }
  int rc = rp_comm_check(c);
  if (rc) fprintf(stderr, "rank %d: rp_comm_check -> %d: %s\n", rank, rc, rp_last_error());
  bar.wait();  // no rank tears down while a peer may still use its region
  rp_comm_destroy(c);
  cudaFree(x);
  cudaFree(y);
  cudaFreeHost(hx);
  cudaFreeHost(hy);
  cudaStreamDestroy(s);
  *bad_out = bad + (rc ? 1 : 0);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  const int W = argc > 1 ? atoi(argv[1]) : 2;
  const int nops = argc > 2 ? atoi(argv[2]) : 40;
  const uint32_t seed = argc > 3 ? (uint32_t)atoi(argv[3]) : 1;
  std::mt19937 g(seed);
  const size_t sizes[] = {1, 7, 1000, 4097, 65536, 203530, 262144, 3u << 20};
  std::vector<Op> ops;
  for (int i = 0; i < nops; ++i) ops.push_back({(int)(g() % 4), sizes[g() % 8], (int)(g() % W)});
  Barrier bar(W);
  std::vector<std::string> blobs(W);
  std::vector<long> bad(W, 0);
  std::vector<int> rcs(W, 0);
  std::vector<std::thread> th;
  for (int r = 0; r < W; ++r)
    th.emplace_back([&, r] { rcs[r] = rank_main(r, W, ops, seed, bar, blobs, &bad[r]); });
  for (auto& t : th) t.join();
  long tot = 0;
  int fail = 0;
  for (int r = 0; r < W; ++r) {
    tot += bad[r];
    fail |= rcs[r];
  }
  printf("lb_abi W=%d ops=%d seed=%u: %s (%ld mismatching elements)\n", W, nops, seed,
         (tot == 0 && !fail) ? "OK" : "FAILED", tot);
  return (tot == 0 && !fail) ? 0 : 1;
}
