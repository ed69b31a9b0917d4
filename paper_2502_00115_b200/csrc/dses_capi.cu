// dses_capi.cu -- host runtime and C ABI (include/dses_b200.h) of the B200 DSES path.
//
// The host side of a registration is native: plan construction (validation of
// what the kernels rely on, fixed-point scaling, spatial tiling of both clouds,
// dedup near lists, device uploads), stage orchestration with CUDA events, and
// the small host<->device scalar traffic between stages.  The Python layer
// (paper_2502_00115_b200/engines.py) mirrors gridreg's API and exceptions on top.
#include <algorithm>
#include <new>
#include <stdexcept>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <cstring>
#include <future>
#include <functional>
#include <deque>
#include <condition_variable>
#include <limits>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/dses_b200.h"
#include "dses_common.cuh"

#ifndef DSES_NVCC_VERSION
#define DSES_NVCC_VERSION "unknown"
#endif

namespace dses {
// dses_vote.cu
cudaError_t launch_vote(const VoteParams& p, bool hsmem, bool psmem, int grid, int threads,
                        cudaStream_t stream);
int vote_max_ctas_per_sm(const VoteParams& p, bool hsmem, bool psmem, int threads);
size_t vote_smem_bytes(const VoteParams& p, bool hsmem, bool psmem, int threads);
size_t vote_static_smem();
cudaError_t launch_vote_blocks(const VoteParams& p, int grid, int threads, cudaStream_t stream);
cudaError_t launch_vote_redo(const VoteParams& p, int grid, int threads, cudaStream_t stream);
// dses_sparse.cu
size_t sparse_scratch_bytes(int64_t n, int64_t m);
cudaError_t launch_sparse_modes(const SparseParams& s, int64_t r_begin, int64_t r_count,
                                void* scratch, size_t scratch_bytes, unsigned long long* counters,
                                int* counts, long long* lins, int* ties, int sms, cudaStream_t st);
cudaError_t launch_narrow_lins(const long long* in, int* out, int64_t n, int sms, cudaStream_t st);
cudaError_t launch_sparse_histogram(const SparseParams& s, bool dedup, void* scratch,
                                    size_t scratch_bytes, unsigned long long* counter,
                                    unsigned long long** out_lins, int** out_counts, int** out_n,
                                    unsigned long long* nkeys_host, int sms, cudaStream_t st);
// dses_score.cu
cudaError_t launch_select_stats(const int* counts, int64_t nrot, unsigned long long* mstar,
                                unsigned long long* nvalid, int sms, cudaStream_t st);
cudaError_t launch_argmax(const int* counts, int64_t nrot, int64_t r_begin, int mstar,
                          unsigned long long* row, int sms, cudaStream_t st,
                          const unsigned long long* dmstar = nullptr);
cudaError_t launch_compact(const int* counts, const int* lins, int64_t nrot, int64_t r_begin,
                           double cutoff, int64_t* rows, int* cl, unsigned long long* ncand, int sms,
                           cudaStream_t st, const unsigned long long* dmstar = nullptr,
                           double q = 0.0);
cudaError_t launch_screen(const ScoreParams& s, const int64_t* rows, const int* lins, int64_t ncand,
                          double* partial, double* err, unsigned long long* minbits, cudaStream_t st,
                          const unsigned long long* dcount = nullptr);
cudaError_t launch_rescore_compact(const double* err, int64_t ncand, double thr, int* sel,
                                   unsigned long long* nsel, cudaStream_t st,
                                   const unsigned long long* dcount = nullptr,
                                   const unsigned long long* dmin = nullptr, double tol = 0.0);
cudaError_t launch_exact(const ScoreParams& s, const int64_t* rows, const int* lins, const int* sel,
                         int64_t nsel, double* vals, double* out, cudaStream_t st,
                         const unsigned long long* dcount = nullptr);
cudaError_t launch_winner(const double* err64, const int* sel, const int64_t* rows, int64_t nsel,
                          double* best_err, int64_t* best_row, int* best_c, cudaStream_t st,
                          const int* lins = nullptr, const unsigned long long* dcount = nullptr);
cudaError_t launch_enumerate_poses(int64_t p0, int64_t np, int64_t ntrans, int64_t* rows, int* lins,
                                   cudaStream_t st);
cudaError_t launch_pick_argmax(const unsigned long long* row, const int* lins, int64_t r_begin,
                               int64_t* cand_rows, int* cand_lins, int* win_c, cudaStream_t st);
cudaError_t launch_finalize(const unsigned long long* scal, const double* win_err, const int* win_c,
                            const int64_t* cand_rows, const int* cand_lins, const int* counts,
                            int64_t r_begin, const double* miss, unsigned long long* stats,
                            long long* rec, cudaStream_t st);
int screen_threads();
int exact_threads();
}  // namespace dses

using namespace dses;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(e_ == cudaErrorMemoryAllocation ? DSES_E_NOMEM : DSES_E_CUDA,           \
                  "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

#define CK_STATUS(call)              \
  do {                               \
    const int s_ = (call);           \
    if (s_ != DSES_OK) return s_;    \
  } while (0)

extern "C" const char* dses_last_error(void) { return g_err.c_str(); }

namespace dses {
// Error reporting for entry points defined in other translation units.
int api_fail(int code, const char* what) { return fail(code, "%s", what); }
}  // namespace dses

extern "C" const char* dses_build_info(void) {
  return "dses_b200: sm_100a, nvcc " DSES_NVCC_VERSION ", fixed-point vote + fp32 screen + fp64 exact";
}

extern "C" int dses_device_count(int* out) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) { *out = 0; return fail(DSES_E_NODEVICE, "%s", cudaGetErrorString(e)); }
  *out = n;
  return DSES_OK;
}

extern "C" int dses_stream_create(int device, void** out) {
  if (!out) return fail(DSES_E_INVALID, "out is NULL");
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n)
    return fail(DSES_E_NODEVICE, "bad device %d", device);
  CK(cudaSetDevice(device));
  cudaStream_t s = nullptr;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *out = (void*)s;
  return DSES_OK;
}

extern "C" int dses_stream_destroy(void* stream) {
  if (!stream) return DSES_OK;
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  CK(cudaStreamDestroy((cudaStream_t)stream));
  return DSES_OK;
}

// ---------------------------------------------------------------------------
// device buffers
// ---------------------------------------------------------------------------
// Device buffers come from the device's stream-ordered memory pool
// (cudaMallocAsync on the legacy stream, release threshold = unlimited), so
// a registration that creates a fresh plan reuses cached memory instead of
// paying cudaMalloc/cudaFree device synchronisations.
static void keep_pool(int device) {
  static std::atomic<bool> done[64];
  if (device < 0 || device >= 64 || done[device].exchange(true)) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    // a plan built on the upload stream must not wait for memory freed behind
    // a search still running on another stream (the pool grows instead)
    int no = 0;
    cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no);
  }
}

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  bool borrowed = false;  // points into another buffer (an upload arena): never freed here
  // A growing buffer is freed and re-allocated on the stream that uses it, so
  // the free is ordered after the work already queued there on the old one.
  // (grow = false: exactly `bytes`, for buffers sized once, e.g. the block lists)
  cudaError_t ensure(size_t bytes, cudaStream_t st, bool grow = true) {
    if (bytes <= cap && p) return cudaSuccess;
    if (p && !borrowed) cudaFreeAsync(p, st);
    p = nullptr;
    cap = 0;
    borrowed = false;
    size_t want = std::max<size_t>(grow ? bytes + bytes / 2 : bytes, 256);
    cudaError_t e = cudaMallocAsync(&p, want, st);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void borrow(void* q, size_t bytes) { release(); p = q; cap = bytes; borrowed = true; }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
  void release() {
    if (p && !borrowed) cudaFreeAsync(p, 0);
    p = nullptr;
    cap = 0;
    borrowed = false;
  }
};

// host<->device traffic is counted per plan (bench.py reports it as e2e bytes)
struct Traffic {
  int64_t h2d = 0, d2h = 0, launches = 0;
};
static thread_local Traffic* g_traffic = nullptr;

static cudaError_t h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (g_traffic) g_traffic->h2d += (int64_t)bytes;
  return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
}
static cudaError_t d2h(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (g_traffic) g_traffic->d2h += (int64_t)bytes;
  return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st);
}
static inline cudaError_t launched(cudaError_t e, int n = 1) {
  if (g_traffic) g_traffic->launches += n;
  return e;
}


// All of a plan's read-only inputs go to the device in ONE copy: packed into
// a per-thread pinned staging buffer, copied into one arena, and the plan's
// buffers borrow sub-ranges of the arena (16 pageable copies cost ~0.2 ms).
struct UploadPack {
  struct Item { DevBuf* buf; const void* src; size_t off, bytes; };
  std::vector<Item> items;
  size_t total = 0;
  template <class T> void add(DevBuf& b, const std::vector<T>& v) {
    const size_t bytes = sizeof(T) * std::max<size_t>(v.size(), 1);
    const size_t off = (total + 255) & ~size_t(255);
    items.push_back({&b, v.empty() ? nullptr : v.data(), off, sizeof(T) * v.size()});
    (void)bytes;
    total = off + bytes;
  }
  // the caller synchronises `st` before the staging buffer is reused
  cudaError_t commit(DevBuf& arena, cudaStream_t st) {
    static thread_local void* staging = nullptr;
    static thread_local size_t staging_cap = 0;
    if (total > staging_cap) {
      if (staging) cudaFreeHost(staging);
      staging = nullptr;
      staging_cap = 0;
      const size_t want = std::max<size_t>(total + total / 2, 1 << 16);
      cudaError_t e = cudaHostAlloc(&staging, want, cudaHostAllocDefault);
      if (e != cudaSuccess) return e;
      staging_cap = want;
    }
    for (const Item& it : items)
      if (it.bytes) std::memcpy(static_cast<unsigned char*>(staging) + it.off, it.src, it.bytes);
    cudaError_t e = arena.ensure(total, st);
    if (e != cudaSuccess) return e;
    e = h2d(arena.p, staging, total, st);
    if (e != cudaSuccess) return e;
    for (const Item& it : items)
      it.buf->borrow(static_cast<unsigned char*>(arena.p) + it.off, it.bytes);
    return cudaSuccess;
  }
};

// ---------------------------------------------------------------------------
// the plan
// ---------------------------------------------------------------------------
namespace {
struct RefTopo;
struct DeviceRef;
struct DeviceFixed;
}  // namespace
struct dses_plan {
  int device = 0, sms = 0;
  std::shared_ptr<const RefTopo> topo;  // the reference cloud's cached topology
  std::shared_ptr<DeviceRef> dref;      // and its device copy (shared by plans)
  std::shared_ptr<DeviceFixed> dfix;    // the fixed-point reference layout on the device (shared)
  size_t smem_optin = 0;
  int64_t n = 0, m = 0, m_pad = 0;
  double bin = 0, inv_bin = 0;
  int64_t ilo[3] = {0, 0, 0}, dims[3] = {1, 1, 1};
  int F = 0;
  int64_t near_pairs = 0;
  double bx = 0, by = 0;             // max |p| bound (|x|_2 + |t|) and max |y| (screen error bound)
  VoteParams vp{};
  bool hsmem = true, psmem = true;
  int vote_grid = 0, vote_threads = kVoteThreads;
  int vote_grid_cap = 0;                               // testing hook: 0 = one wave
  int blk_s[3] = {0, 0, 0};                            // rotation-block sides (0: per-rotation kernel)
  int blk_cap = kBlockListCap;                         // list entries per CTA (testing hook)
  double lane_use = 0;                                 // estimated lane use of the per-rotation kernel
  DevBuf blist, redo;                                  // block kernel: candidate lists, redo rotations
  // device data
  DevBuf xs, ys, yq, near_off, near_idx, xt, yt;  // vote (tile order)
  DevBuf risk;                                         // vote: guard-band risk bitmaps per group
  DevBuf x0, ys0, ys1, ys2, ysf;                      // scoring (original x, y sorted by axis 0)
  DevBuf gcell, gpts;                                  // scoring: uniform grid over y
  DevBuf arena;                                        // the inputs above live here (UploadPack)
  DevBuf yorig;                                        // (m, 3) reference, original order (sparse path)
  bool sparse = false;                                 // lattice beyond kDenseMaxBins: sort-based mode
  DevBuf lins64, sparse_scratch;
  float gorg[3] = {0, 0, 0}, gh = 1.f, g_pts_per_cell = 1.f;
  int gdim[3] = {1, 1, 1};
  DevBuf cth, sth, rots;                               // rotation sources
  DevBuf counts, lins, ties;                           // per-rotation outputs
  DevBuf hist_g, p_g;                                  // global fallbacks
  DevBuf stats, scal;                                  // counters / scalar outputs
  DevBuf cand_rows, cand_lins, err32, partial, sel, vals, err64;
  DevBuf win_err, win_row, win_c, tmp_rows, tmp_lins, tvec;
  // stage state
  int64_t cur_r_begin = 0, cur_r_count = 0, cur_k = 0;
  RotSource cur_rot{};
  int64_t kept = 0;
  cudaEvent_t ev[8];
  Traffic traffic;       // counters since the last dses_stage_stats / dses_search
  bool vote_timed = false;
  long long* rec_host = nullptr;  // pinned result record of dses_search (12 slots)
  struct Pending {                // a dses_search_async awaiting dses_search_wait
    bool active = false;
    dses_grid g{};
    int64_t r_begin = 0, r_count = 0, cap = 0;
    double q = 0, param = 0;
    int code = 0, skip_refine = 0;
    void* stream = nullptr;
  } pend;
};

// Pinned 128-byte result records, carved from page-locked slabs (one
// cudaHostAlloc per 256 plans instead of one per plan).
static std::mutex g_rec_mu;
static std::vector<long long*> g_rec_free;
static long long* rec_take() {
  std::lock_guard<std::mutex> lk(g_rec_mu);
  if (g_rec_free.empty()) {
    void* slab = nullptr;
    if (cudaHostAlloc(&slab, 256 * 128, cudaHostAllocPortable) != cudaSuccess) return nullptr;
    for (int k = 255; k >= 0; --k)
      g_rec_free.push_back(reinterpret_cast<long long*>(static_cast<char*>(slab) + 128 * k));
  }
  long long* r = g_rec_free.back();
  g_rec_free.pop_back();
  return r;
}
static void rec_give(long long* r) {
  if (!r) return;
  std::lock_guard<std::mutex> lk(g_rec_mu);
  g_rec_free.push_back(r);
}

// Plan construction uploads on a non-blocking stream of the calling thread,
// so building the next registration's plan never waits for a search running
// on the caller's stream.
static cudaStream_t upload_stream(int device) {
  static thread_local cudaStream_t streams[64] = {};
  if (device < 0 || device >= 64) return 0;
  if (!streams[device]) cudaStreamCreateWithFlags(&streams[device], cudaStreamNonBlocking);
  return streams[device];
}

// RAII: route the copy/launch counters of this call to the plan
struct TrafficScope {
  Traffic* prev;
  explicit TrafficScope(dses_plan* P) : prev(g_traffic) { g_traffic = P ? &P->traffic : nullptr; }
  ~TrafficScope() { g_traffic = prev; }
};

namespace {

// DSES_TRACE=1 prints the plan-construction steps to stderr (debug aid)
void trace(const char* what) {
  static const int on = [] { const char* e = getenv("DSES_TRACE"); return e && *e == '1'; }();
  if (on) {
    static auto t0 = std::chrono::steady_clock::now();
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    fprintf(stderr, "[dses %10.3f ms] %s\n", ms, what);
    fflush(stderr);
  }
}

// round-half-away-from-zero integer of v (host side fixed-point conversion)
inline int64_t rint64(double v) { return (int64_t)std::llrint(v); }

struct KdPoint {  // a point with its index, contiguous for the median splits
  double c[3];
  int idx;
};

static void kd_split(KdPoint* a, int64_t lo, int64_t hi, std::vector<std::pair<int, int>>& tiles,
                     int tile, int spawn) {
  const int64_t cnt = hi - lo;
  if (cnt <= tile) {
    if (cnt > 0) tiles.emplace_back((int)lo, (int)cnt);
    return;
  }
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t q = lo; q < hi; ++q)
    for (int k = 0; k < 3; ++k) {
      mn[k] = std::min(mn[k], a[q].c[k]);
      mx[k] = std::max(mx[k], a[q].c[k]);
    }
  int axis = 0;
  for (int k = 1; k < 3; ++k)
    if (mx[k] - mn[k] > mx[axis] - mn[axis]) axis = k;
  const int64_t ntile = (cnt + tile - 1) / tile;
  const int64_t left = (ntile / 2) * tile;
  std::nth_element(a + lo, a + lo + left, a + hi, [axis](const KdPoint& u, const KdPoint& v) {
    return u.c[axis] < v.c[axis] || (u.c[axis] == v.c[axis] && u.idx < v.idx);
  });
  if (spawn > 0 && cnt >= 32768) {  // disjoint halves: left on a helper thread
    std::vector<std::pair<int, int>> lt, rt;
    std::thread th([&] { kd_split(a, lo, lo + left, lt, tile, spawn - 1); });
    kd_split(a, lo + left, hi, rt, tile, spawn - 1);
    th.join();
    tiles.insert(tiles.end(), lt.begin(), lt.end());
    tiles.insert(tiles.end(), rt.begin(), rt.end());
    return;
  }
  kd_split(a, lo, lo + left, tiles, tile, 0);
  kd_split(a, lo + left, hi, tiles, tile, 0);
}

// Persistent helper threads for the host-side plan build (thread creation
// costs about as much as the work it would take over for clouds of a few
// thousand points).
class HelperPool {
 public:
  explicit HelperPool(int n) {
    for (int i = 0; i < n; ++i) th_.emplace_back([this] { loop(); });
  }
  ~HelperPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  std::future<void> submit(std::function<void()> fn) {
    auto task = std::make_shared<std::packaged_task<void()>>(std::move(fn));
    std::future<void> f = task->get_future();
    {
      std::lock_guard<std::mutex> lk(mu_);
      q_.push_back([task] { (*task)(); });
    }
    cv_.notify_one();
    return f;
  }
 private:
  void loop() {
    for (;;) {
      std::function<void()> job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [this] { return stop_ || !q_.empty(); });
        if (stop_ && q_.empty()) return;
        job = std::move(q_.front());
        q_.pop_front();
      }
      job();
    }
  }
  std::vector<std::thread> th_;
  std::deque<std::function<void()>> q_;
  std::mutex mu_;
  std::condition_variable cv_;
  bool stop_ = false;
};

static HelperPool& helper_pool() {
  static HelperPool pool(3);
  return pool;
}

// Recursive median split of pts[perm[lo..hi)] until tiles hold <= `tile`
// points; splits at a multiple of `tile` so that all but the last tile of
// each branch are full.  perm is reordered into tile order.  Clouds of
// >= 2048 points: the first two levels on this thread, the four subtrees on
// it and three persistent helpers (disjoint ranges, tiles in order).
void kd_tiles(const double* pts, int64_t lo, int64_t hi, std::vector<int>& perm,
              std::vector<std::pair<int, int>>& tiles, int tile, int spawn = 0) {
  std::vector<KdPoint> a((size_t)(hi - lo));
  for (int64_t q = lo; q < hi; ++q) {
    KdPoint& k = a[(size_t)(q - lo)];
    k.idx = perm[q];
    for (int d = 0; d < 3; ++d) k.c[d] = pts[3 * (int64_t)k.idx + d];
  }
  std::vector<std::pair<int, int>> t;
  if (spawn > 0 && hi - lo >= 2048) {
    // two median levels here: up to four disjoint subranges
    std::vector<std::pair<int64_t, int64_t>> r1, r2;
    auto split = [&](int64_t l, int64_t h, std::vector<std::pair<int64_t, int64_t>>& out) {
      const int64_t cnt = h - l;
      if (cnt <= tile) { out.emplace_back(l, h); return; }
      double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
      for (int64_t q = l; q < h; ++q)
        for (int k = 0; k < 3; ++k) {
          mn[k] = std::min(mn[k], a[q].c[k]);
          mx[k] = std::max(mx[k], a[q].c[k]);
        }
      int axis = 0;
      for (int k = 1; k < 3; ++k)
        if (mx[k] - mn[k] > mx[axis] - mn[axis]) axis = k;
      const int64_t left = (((cnt + tile - 1) / tile) / 2) * tile;
      std::nth_element(a.begin() + l, a.begin() + l + left, a.begin() + h,
                       [axis](const KdPoint& u, const KdPoint& v) {
                         return u.c[axis] < v.c[axis] || (u.c[axis] == v.c[axis] && u.idx < v.idx);
                       });
      out.emplace_back(l, l + left);
      out.emplace_back(l + left, h);
    };
    split(0, hi - lo, r1);
    for (const auto& r : r1) split(r.first, r.second, r2);
    std::vector<std::vector<std::pair<int, int>>> parts(r2.size());
    std::vector<std::future<void>> fut;
    for (size_t k = 1; k < r2.size(); ++k)
      fut.push_back(helper_pool().submit([&, k] { kd_split(a.data(), r2[k].first, r2[k].second, parts[k], tile, 0); }));
    kd_split(a.data(), r2[0].first, r2[0].second, parts[0], tile, 0);
    for (auto& f : fut) f.get();
    for (const auto& pt : parts) t.insert(t.end(), pt.begin(), pt.end());
  } else {
    kd_split(a.data(), 0, hi - lo, t, tile, 0);
  }
  for (int64_t q = lo; q < hi; ++q) perm[q] = a[(size_t)(q - lo)].idx;
  for (const auto& e : t) tiles.emplace_back(e.first + (int)lo, e.second);
}

// Like kd_tiles for weighted items (centroids cen, weights wt >= 1): leaves
// hold items of total weight <= cap.  Median splits by item count
// (nth_element, O(n) per level) placed so that the left part holds about
// floor(leaves / 2) * cap weight; a leaf that ends up over capacity is simply
// split again.
void kd_weighted(const double* cen, const std::vector<int>& wt, int64_t lo, int64_t hi,
                 std::vector<int>& perm, std::vector<std::pair<int, int>>& tiles, int cap,
                 int64_t leaves, int spawn = 0) {
  int64_t W = 0;
  for (int64_t q = lo; q < hi; ++q) W += wt[perm[q]];
  leaves = std::max<int64_t>(leaves, (W + cap - 1) / cap);
  if (leaves <= 1 || hi - lo <= 1) {
    if (hi > lo) tiles.emplace_back((int)lo, (int)(hi - lo));
    return;
  }
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t q = lo; q < hi; ++q)
    for (int k = 0; k < 3; ++k) {
      mn[k] = std::min(mn[k], cen[3 * perm[q] + k]);
      mx[k] = std::max(mx[k], cen[3 * perm[q] + k]);
    }
  int axis = 0;
  for (int k = 1; k < 3; ++k)
    if (mx[k] - mn[k] > mx[axis] - mn[axis]) axis = k;
  // the left part gets half the leaf budget and the same share of the weight,
  // so both parts keep the parent's fill fraction (slack is spread evenly
  // instead of spilling one item into an extra, nearly empty leaf).
  const int64_t lleaves = leaves / 2;
  const int64_t target = std::max<int64_t>(1, W * lleaves / leaves);
  // split index s: the left part (the s - lo smallest along `axis`) carries as
  // close to `target` weight as the item weights allow without exceeding it.
  // nth_element partitions in O(n); a few corrections settle s.
  auto less = [&](int a, int b) {
    const double va = cen[3 * a + axis], vb = cen[3 * b + axis];
    return va < vb || (va == vb && a < b);
  };
  int64_t s = lo + (int64_t)((double)target * (double)(hi - lo) / (double)W);
  s = std::min(hi - 1, std::max(lo + 1, s));
  std::nth_element(perm.begin() + lo, perm.begin() + s, perm.begin() + hi, less);
  int64_t wl = 0;
  for (int64_t q = lo; q < s; ++q) wl += wt[perm[q]];
  if (wl > target) {  // hand the largest left items to the right part
    const int64_t k = std::min<int64_t>(s - lo - 1, wl - target);
    std::nth_element(perm.begin() + lo, perm.begin() + (s - k), perm.begin() + s, less);
    std::sort(perm.begin() + (s - k), perm.begin() + s, less);
    while (wl > target && s > lo + 1) wl -= wt[perm[--s]];
  } else if (wl < target) {  // take the smallest right items while they fit
    const int64_t k = std::min<int64_t>(hi - s - 1, target - wl);
    if (k > 0) {
      std::nth_element(perm.begin() + s, perm.begin() + (s + k), perm.begin() + hi, less);
      std::sort(perm.begin() + s, perm.begin() + (s + k), less);
      while (s < hi - 1 && s < s + k && wl + wt[perm[s]] <= target) wl += wt[perm[s++]];
    }
  }
  if (spawn > 0 && hi - lo >= 4096) {  // disjoint halves: left on a helper thread
    std::vector<std::pair<int, int>> left;
    std::thread th([&] { kd_weighted(cen, wt, lo, s, perm, left, cap, lleaves, spawn - 1); });
    std::vector<std::pair<int, int>> right;
    kd_weighted(cen, wt, s, hi, perm, right, cap, leaves - lleaves, spawn - 1);
    th.join();
    tiles.insert(tiles.end(), left.begin(), left.end());
    tiles.insert(tiles.end(), right.begin(), right.end());
    return;
  }
  kd_weighted(cen, wt, lo, s, perm, tiles, cap, lleaves);
  kd_weighted(cen, wt, s, hi, perm, tiles, cap, leaves - lleaves);
}

// Unordered pairs (a, b), a != b, of reference points closer than thr in
// every axis.  Points are bucketed into strips of width thr along axis 0 and
// sorted by axis 1 inside each strip; a point's partners lie in its own strip
// (later in axis-1 order) or in the next strip (an axis-1 window found by
// binary search), so each pair is found once.
// host threads for plan construction of large clouds (at most 8)
static int host_threads() {
  static const int n = [] {
    const unsigned h = std::thread::hardware_concurrency();
    return (int)std::max(1u, std::min(8u, h));
  }();
  return n;
}

std::vector<std::pair<int, int>> near_pairs(const double* y, int64_t m, double thr) {
  double mn0 = INFINITY;
  for (int64_t j = 0; j < m; ++j) mn0 = std::min(mn0, y[3 * j]);
  const double width = thr * (1.0 + 1e-9);  // partners are never two strips apart
  struct Key { int64_t strip; double y1; int idx; };
  auto by_y1 = [](const Key& a, const Key& b) {
    return a.y1 < b.y1 || (a.y1 == b.y1 && a.idx < b.idx);
  };
  std::vector<Key> keys(m);
  int64_t smax = 0;
  for (int64_t j = 0; j < m; ++j) {
    keys[j] = {(int64_t)std::floor((y[3 * j] - mn0) / width), y[3 * j + 1], (int)j};
    smax = std::max(smax, keys[j].strip);
  }
  if (smax <= 4 * m + 1024) {
    // counting sort by strip, then each strip by (y1, index) -- strips over
    // host threads for large clouds
    std::vector<int64_t> so(smax + 2, 0);
    for (const Key& k : keys) ++so[k.strip + 1];
    for (int64_t t = 0; t <= smax; ++t) so[t + 1] += so[t];
    std::vector<Key> sorted(m);
    {
      std::vector<int64_t> fill(so.begin(), so.end() - 1);
      for (const Key& k : keys) sorted[fill[k.strip]++] = k;
    }
    keys.swap(sorted);
    auto sort_strips = [&](int64_t t0, int64_t t1) {
      for (int64_t t = t0; t < t1; ++t)
        if (so[t + 1] - so[t] > 1) std::sort(keys.begin() + so[t], keys.begin() + so[t + 1], by_y1);
    };
    const int nt = m >= 8192 ? host_threads() : 1;
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t)
      pool.emplace_back(sort_strips, (smax + 1) * t / nt, (smax + 1) * (t + 1) / nt);
    sort_strips(0, (smax + 1) / nt);
    for (auto& th : pool) th.join();
  } else {
    std::sort(keys.begin(), keys.end(), [&](const Key& a, const Key& b) {
      return a.strip != b.strip ? a.strip < b.strip : by_y1(a, b);
    });
  }
  auto close = [&](int a, int b) {
    return std::fabs(y[3 * a] - y[3 * b]) < thr && std::fabs(y[3 * a + 1] - y[3 * b + 1]) < thr &&
           std::fabs(y[3 * a + 2] - y[3 * b + 2]) < thr;
  };
  // strips [p, e) scanned against themselves and the next strip; large
  // clouds split the key range at strip boundaries over host threads and
  // concatenate in key order (the same pair order as one thread)
  auto scan = [&](int64_t p, int64_t end, std::vector<std::pair<int, int>>& out) {
    while (p < end) {
      const int64_t sp = keys[p].strip;
      int64_t e = p;
      while (e < m && keys[e].strip == sp) ++e;  // current strip [p, e)
      int64_t ne = e;
      while (ne < m && keys[ne].strip == sp + 1) ++ne;  // next strip [e, ne)
      for (int64_t q = p; q < e; ++q) {
        const int a = keys[q].idx;
        const double y1 = keys[q].y1;
        for (int64_t r = q + 1; r < e && keys[r].y1 - y1 < thr; ++r)
          if (close(a, keys[r].idx)) out.emplace_back(a, keys[r].idx);
        int64_t lo = e, hi2 = ne;  // next strip: axis-1 window (y1 - thr, y1 + thr)
        while (lo < hi2) {
          const int64_t mid = (lo + hi2) / 2;
          if (keys[mid].y1 <= y1 - thr) lo = mid + 1; else hi2 = mid;
        }
        for (int64_t r = lo; r < ne && keys[r].y1 - y1 < thr; ++r)
          if (close(a, keys[r].idx)) out.emplace_back(a, keys[r].idx);
      }
      p = e;
    }
  };
  const int nt = m >= 8192 ? host_threads() : 1;
  std::vector<int64_t> cut(nt + 1, m);
  cut[0] = 0;
  for (int t = 1; t < nt; ++t) {  // chunk starts moved forward to a strip boundary
    int64_t c = std::max(cut[t - 1], m * t / nt);
    while (c > 0 && c < m && keys[c].strip == keys[c - 1].strip) ++c;
    cut[t] = c;
  }
  std::vector<std::vector<std::pair<int, int>>> parts(nt);
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(scan, cut[t], cut[t + 1], std::ref(parts[t]));
  scan(cut[0], cut[1], parts[0]);
  for (auto& th : pool) th.join();
  std::vector<std::pair<int, int>> out = std::move(parts[0]);
  for (int t = 1; t < nt; ++t) out.insert(out.end(), parts[t].begin(), parts[t].end());
  return out;
}

// ---------------------------------------------------------------------------
// Reference-cloud topology: everything of a plan that depends only on the
// reference cloud and the bin size -- the scoring layout (axis-0 sort, fp32
// copy, uniform grid), the dedup partners (points closer than one bin per
// axis), their components, the reference groups (k-d tiles over the
// components) and the exact path's near lists.  Cached for the most recent
// clouds (content-compared), so registering many sources against one model
// (the c4 tool-pose use) builds it once.
// ---------------------------------------------------------------------------
struct GroupSpan { int start, count, gm; };
struct RefFixed;
struct RefTopo {
  int64_t m = 0;
  double bin = 0;
  std::vector<double> y;                       // the cloud (cache key, compared exactly)
  std::vector<double> c0, c1, c2;              // axis-0-sorted columns
  std::vector<float4> yf, gp;                  // fp32 copy; grid-ordered points
  std::vector<int2> range;                     // grid cells
  float gorg[3] = {0, 0, 0}, gh = 1.f, gppc = 1.f;
  int gdim[3] = {1, 1, 1};
  std::vector<std::pair<int, int>> near;       // dedup partner pairs
  std::vector<int> aoff, aidx;                 // their adjacency (CSR, original indices)
  std::vector<int> yidx;                       // tile-order entry -> original index
  std::vector<char> yfar;                      // component too large for a warp
  std::vector<int> ycomp;                      // tile-order entry of its component's first point
  std::vector<GroupSpan> groups;
  std::vector<int> pos;                        // original index -> tile-order entry
  std::vector<int> noff, nidx;                 // exact-path near lists (tile order, j' < j)
  std::vector<double> ys;                      // the cloud in tile order
  double ymax = 0, ext = 0;                    // max |y| over the axes; largest axis extent
  std::vector<double> gbox;                    // per reference group: lo xyz, hi xyz (world)
  mutable std::mutex dmu;
  mutable std::shared_ptr<DeviceRef> dev[64];  // device copies of the arrays above
  mutable std::mutex fmu;
  mutable std::vector<std::shared_ptr<const RefFixed>> fixed;  // fixed-point layouts (ref_fixed)
};

// A RefTopo's read-only arrays on one device, uploaded once and borrowed by
// every plan of that reference cloud (freed with the last plan / eviction).
struct DeviceRef {
  int device = 0;
  DevBuf arena, yorig, ys, near_off, near_idx, ys0, ys1, ys2, ysf, gcell, gpts;
  ~DeviceRef() {  // possibly on another thread's current device (cache eviction)
    if (!arena.p) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    cudaFree(arena.p);  // synchronous: no plan of this cloud is left
    cudaSetDevice(cur);
    arena.p = nullptr;
  }
};

static std::shared_ptr<const RefTopo> build_ref_topo(const double* y, int64_t m, double bin) {
  auto T = std::make_shared<RefTopo>();
  T->m = m;
  T->bin = bin;
  T->y.assign(y, y + 3 * m);
  std::vector<double>& c0 = T->c0; std::vector<double>& c1 = T->c1; std::vector<double>& c2 = T->c2;
  std::vector<float4>& yf = T->yf; std::vector<float4>& gp = T->gp;
  std::vector<int2>& range = T->range;
  RefTopo* PT = T.get();
  // ---- scoring layout (y sorted by axis 0, fp32 copy, uniform grid) on a
  //      persistent helper thread: independent of the vote layout built below
  auto scoring = helper_pool().submit([&]() {
  // ---- scoring layout: x original order, y sorted by axis 0 (stable)
  trace("scoring layout");
  std::vector<int> sy(m);
  {  // stable sort by axis 0 == sort by (y0, index)
    std::vector<std::pair<double, int>> k0(m);
    for (int64_t j = 0; j < m; ++j) k0[j] = {y[3 * j], (int)j};
    std::sort(k0.begin(), k0.end());
    for (int64_t j = 0; j < m; ++j) sy[j] = k0[j].second;
  }
  c0.resize(m); c1.resize(m); c2.resize(m);
  yf.resize(m);
  for (int64_t j = 0; j < m; ++j) {
    c0[j] = y[3 * sy[j]];
    c1[j] = y[3 * sy[j] + 1];
    c2[j] = y[3 * sy[j] + 2];
    yf[j] = make_float4((float)c0[j], (float)c1[j], (float)c2[j], 0.f);
  }
  {  // uniform grid over y for the screen's nearest-neighbour search: cells of
     // 4 translation bins (grown until the grid has <= 2^20 cells)
    trace("score grid");
    float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t j = 0; j < m; ++j)
      for (int k = 0; k < 3; ++k) {
        const float v = (&yf[j].x)[k];
        mn[k] = std::min(mn[k], v);
        mx[k] = std::max(mx[k], v);
      }
    double h = 4.0 * bin;
    int dim[3];
    for (;;) {
      int64_t cells = 1;
      for (int k = 0; k < 3; ++k) {
        dim[k] = (int)std::min<double>(std::floor((mx[k] - mn[k]) / h) + 1.0, 1 << 20);
        cells *= dim[k];
      }
      if (cells <= (1 << 20)) break;
      h *= 1.25;
    }
    const float hf = (float)h, inv = (float)(1.0 / h);
    auto cell_of = [&](const float4& q) {
      int c[3];
      for (int k = 0; k < 3; ++k)
        c[k] = std::min(dim[k] - 1, std::max(0, (int)std::floor(((&q.x)[k] - mn[k]) * inv)));
      return (c[0] * dim[1] + c[1]) * dim[2] + c[2];
    };
    const int ncell = dim[0] * dim[1] * dim[2];
    std::vector<int> cnt(ncell + 1, 0), cid(m);
    for (int64_t j = 0; j < m; ++j) { cid[j] = cell_of(yf[j]); ++cnt[cid[j] + 1]; }
    for (int c = 0; c < ncell; ++c) cnt[c + 1] += cnt[c];
    range.resize(ncell);
    for (int c = 0; c < ncell; ++c) range[c] = make_int2(cnt[c], cnt[c + 1]);
    gp.resize(m);
    std::vector<int> fill(cnt.begin(), cnt.end() - 1);
    for (int64_t j = 0; j < m; ++j) {  // .w: the point's index in axis-0 order (exact re-score)
      float4 g = yf[j];
      int jj = (int)j;
      std::memcpy(&g.w, &jj, sizeof jj);
      gp[fill[cid[j]]++] = g;
    }
    int occupied = 0;
    for (int c = 0; c < ncell; ++c) occupied += range[c].y > range[c].x;
    PT->gppc = (float)m / (float)std::max(1, occupied);
    for (int k = 0; k < 3; ++k) { PT->gorg[k] = mn[k]; PT->gdim[k] = dim[k]; }
    PT->gh = hf;
  }
  });
  // ---- reference layout.  Dedup partners (points closer than one bin per
  // axis: the only pairs that can share a bin for one source) form
  // components; groups of <= 32 points (one per lane) are k-d tiles over the
  // components, so that every partner of a point sits in the same warp and
  // the per-source dedup is a lane shuffle.  Points of components larger
  // than kMaxComp, and points with more than two earlier partners, are
  // flagged "far" and take the exact path when they vote.
  trace("dedup components");
  const double thr = bin * (1.0 + 1e-6);
  std::vector<std::pair<int, int>> near_v = near_pairs(y, m, thr);
  const std::vector<std::pair<int, int>>& near = near_v;
  trace("  near pairs");
  // adjacency in CSR form
  std::vector<int> aoff(m + 1, 0), aidx(2 * near.size());
  for (const auto& e : near) { ++aoff[e.first + 1]; ++aoff[e.second + 1]; }
  for (int64_t j = 0; j < m; ++j) aoff[j + 1] += aoff[j];
  {
    std::vector<int> fill(aoff.begin(), aoff.end() - 1);
    for (const auto& e : near) { aidx[fill[e.first]++] = e.second; aidx[fill[e.second]++] = e.first; }
  }
  // components (flat): item q = points ipts[ioff[q] .. ioff[q+1]), sorted
  std::vector<int> ioff(1, 0), ipts;
  std::vector<char> item_far;
  ipts.reserve(m);
  {
    std::vector<char> seen(m, 0);
    std::vector<int> c;
    for (int64_t s0 = 0; s0 < m; ++s0) {
      if (seen[s0]) continue;
      c.assign(1, (int)s0);
      seen[s0] = 1;
      for (size_t h = 0; h < c.size(); ++h)
        for (int a = aoff[c[h]]; a < aoff[c[h] + 1]; ++a)
          if (!seen[aidx[a]]) { seen[aidx[a]] = 1; c.push_back(aidx[a]); }
      if (c.size() > 1) std::sort(c.begin(), c.end());
      if ((int)c.size() <= kMaxComp) {
        ipts.insert(ipts.end(), c.begin(), c.end());
        ioff.push_back((int)ipts.size());
        item_far.push_back(0);
      } else {
        for (int v : c) { ipts.push_back(v); ioff.push_back((int)ipts.size()); item_far.push_back(1); }
      }
    }
  }
  const size_t nitems = item_far.size();
  trace("  components");
  std::vector<double> cen(3 * nitems);
  std::vector<int> wt(nitems);
  for (size_t q = 0; q < nitems; ++q) {
    wt[q] = ioff[q + 1] - ioff[q];
    for (int k = 0; k < 3; ++k) {
      double acc = 0;
      for (int a = ioff[q]; a < ioff[q + 1]; ++a) acc += y[3 * ipts[a] + k];
      cen[3 * q + k] = acc / (double)wt[q];
    }
  }
  std::vector<int> iperm(nitems);
  std::iota(iperm.begin(), iperm.end(), 0);
  std::vector<std::pair<int, int>> itiles;
  // leaf budget = ceil(total / 32); a looser budget (fewer-filled groups) grew
  // the group boxes more than it saved lanes (experiments)
  kd_weighted(cen.data(), wt, 0, (int64_t)nitems, iperm, itiles, kTile, 0,
              host_threads() >= 8 ? 3 : host_threads() >= 4 ? 2 : 0);
  trace("  component k-d tiles");
  std::vector<int>& yidx = T->yidx;
  std::vector<char>& yfar = T->yfar;
  std::vector<GroupSpan>& groups = T->groups;
  std::vector<int>& ycomp = T->ycomp;
  for (const auto& t : itiles) {
    const int start = (int)yidx.size();
    for (int q = t.first; q < t.first + t.second; ++q) {
      const int cfirst = (int)yidx.size();
      for (int a = ioff[iperm[q]]; a < ioff[iperm[q] + 1]; ++a) {
        yidx.push_back(ipts[a]);
        yfar.push_back(item_far[iperm[q]]);
        ycomp.push_back(cfirst);
      }
    }
    groups.push_back({start, (int)yidx.size() - start, 1});
  }
  const int64_t mp = (int64_t)yidx.size();
  std::vector<int>& pos = T->pos;
  pos.assign(m, 0);
  for (int64_t q = 0; q < mp; ++q) pos[yidx[q]] = (int)q;
  // ---- full dedup near lists (tile order, j' < j) for the exact path
  trace("dedup near lists");
  // CSR near lists in tile order: j' < j, sorted (the exact path's partners)
  const int64_t npairs = (int64_t)near.size();
  std::vector<int>& noff = T->noff;
  std::vector<int>& nidx = T->nidx;
  noff.assign(mp + 1, 0);
  nidx.assign((size_t)npairs, 0);
  for (const auto& e : near) ++noff[std::max(pos[e.first], pos[e.second]) + 1];
  for (int64_t q = 0; q < mp; ++q) noff[q + 1] += noff[q];
  {
    std::vector<int> fill(noff.begin(), noff.end() - 1);
    for (const auto& e : near) {
      const int a = pos[e.first], b = pos[e.second];
      nidx[fill[std::max(a, b)]++] = std::min(a, b);
    }
    for (int64_t q = 0; q < mp; ++q)
      if (noff[q + 1] - noff[q] > 1) std::sort(nidx.begin() + noff[q], nidx.begin() + noff[q + 1]);
  }
  T->aoff = std::move(aoff);
  T->aidx = std::move(aidx);
  T->near = std::move(near_v);
  T->ys.resize(3 * mp);
  for (int64_t q = 0; q < mp; ++q)
    for (int k = 0; k < 3; ++k) T->ys[3 * q + k] = y[3 * yidx[q] + k];
  for (int k = 0; k < 3; ++k) {
    double lo = INFINITY, hi = -INFINITY;
    for (int64_t j = 0; j < m; ++j) {
      lo = std::min(lo, y[3 * j + k]);
      hi = std::max(hi, y[3 * j + k]);
      T->ymax = std::max(T->ymax, std::fabs(y[3 * j + k]));
    }
    if (m > 0) T->ext = std::max(T->ext, hi - lo);
  }
  T->gbox.assign(6 * groups.size(), 0.0);
  for (size_t g = 0; g < groups.size(); ++g) {
    double* b = &T->gbox[6 * g];
    for (int k = 0; k < 3; ++k) { b[k] = INFINITY; b[3 + k] = -INFINITY; }
    for (int q = groups[g].start; q < groups[g].start + groups[g].count; ++q)
      for (int k = 0; k < 3; ++k) {
        b[k] = std::min(b[k], T->ys[3 * q + k]);
        b[3 + k] = std::max(b[3 + k], T->ys[3 * q + k]);
      }
  }
  scoring.get();
  return T;
}

static std::shared_ptr<const RefTopo> ref_topo(const double* y, int64_t m, double bin) {
  static std::mutex mu;
  static std::vector<std::shared_ptr<const RefTopo>> cache;  // most recent last
  constexpr size_t kKeep = 4;
  {
    std::lock_guard<std::mutex> lk(mu);
    for (size_t k = cache.size(); k-- > 0;) {
      const auto& c = cache[k];
      if (c->m == m && c->bin == bin && std::memcmp(c->y.data(), y, sizeof(double) * 3 * m) == 0) {
        auto hit = c;
        cache.erase(cache.begin() + (ptrdiff_t)k);
        cache.push_back(hit);
        trace("reference topology: cached");
        return hit;
      }
    }
  }
  auto T = build_ref_topo(y, m, bin);
  std::lock_guard<std::mutex> lk(mu);
  cache.push_back(T);
  if (cache.size() > kKeep) cache.erase(cache.begin());
  return T;
}

// The reference cloud in fixed point for one (F, window origin): Yq in tile
// order (the vote kernels' metadata in .w, the block kernel's empty sentinel
// slot at m_pad), the group tiles and the guard-band risk bitmaps.  Cached per
// reference topology (most recent few) and uploaded once per device, like
// the topology: registrations of many sources against one model with one
// search configuration build it once.
struct DeviceFixed {
  int device = 0;
  DevBuf arena, yq, yt, risk;
  ~DeviceFixed() {
    if (!arena.p) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    cudaFree(arena.p);  // synchronous: no plan of this layout is left
    cudaSetDevice(cur);
    arena.p = nullptr;
  }
};
struct RefFixed {
  int F = 0;
  int64_t ilo[3] = {0, 0, 0};
  std::vector<int4> yq;
  std::vector<YTile> yt;
  std::vector<unsigned> risk;
  bool risk_on = false;
  mutable std::mutex dmu;
  mutable std::shared_ptr<DeviceFixed> dev[64];
};

static int build_ref_fixed(const RefTopo& T, double inv_bin, int F, const int64_t ilo[3], RefFixed* R) {
  R->F = F;
  for (int k = 0; k < 3; ++k) R->ilo[k] = ilo[k];
  const std::vector<int>& yidx = T.yidx;
  const std::vector<char>& yfar = T.yfar;
  const std::vector<GroupSpan>& groups = T.groups;
  const std::vector<int>& aoff = T.aoff;
  const std::vector<int>& aidx = T.aidx;
  const std::vector<int>& pos = T.pos;
  const std::vector<double>& ys = T.ys;
  const int64_t mp = (int64_t)yidx.size();
  const double S = std::ldexp(1.0, F);
  // fixed-point reference: Yq = rint(fl(y*inv)*S) - lo*S + S/2 + G
  std::vector<int4>& yq = R->yq;
  yq.resize(mp);
  const int64_t Si = (int64_t)1 << F;
  for (int64_t q = 0; q < mp; ++q) {
    int v[3];
    for (int k = 0; k < 3; ++k) {
      int64_t w = F ? rint64((ys[3 * q + k] * inv_bin) * S) - ilo[k] * Si + Si / 2 + kGuard : 0;
      if (w > (1ll << 30) || w < -(1ll << 30)) {
        return fail(DSES_E_INVALID, "internal: fixed-point overflow (F=%d)", F);
      }
      v[k] = (int)w;
    }
    yq[q] = make_int4(v[0], v[1], v[2], 0);
  }
  std::vector<YTile>& yt = R->yt;
  yt.resize(groups.size());
  for (size_t t = 0; t < groups.size(); ++t) {
    YTile& T = yt[t];
    T = YTile{};
    T.start = groups[t].start;
    T.count = groups[t].count;
    T.gm = 0;  // max earlier partners resolved by shuffle in this group
    for (int k = 0; k < 3; ++k) { T.lo[k] = INT32_MAX; T.hi[k] = INT32_MIN; }
    for (int q = T.start; q < T.start + T.count; ++q) {
      ++T.npts;
      const int v[3] = {yq[q].x, yq[q].y, yq[q].z};
      for (int k = 0; k < 3; ++k) { T.lo[k] = std::min(T.lo[k], v[k]); T.hi[k] = std::max(T.hi[k], v[k]); }
      // earlier partners (tile order) of point q: lanes of the same group
      int w = 0, ne = 0;
      bool far = yfar[q];
      for (int a = aoff[yidx[q]]; a < aoff[yidx[q] + 1]; ++a) {
        const int q2 = pos[aidx[a]];
        if (q2 >= q) continue;
        if (q2 < T.start || ne == 2) { far = true; continue; }
        w |= (q2 - T.start + 1) << (6 * ne);
        ++ne;
      }
      if (!far) T.gm = std::max(T.gm, ne);
      yq[q].w = far ? kFarFlag : w;
    }
    // unused partner slots (below the group's shuffle count gm) -> a safe
    // lane: an empty lane of the group, else the first non-far point that is
    // no dedup partner of q; a point without one takes the exact path
    if (T.gm > 0) {
      for (int q = T.start; q < T.start + T.count; ++q) {
        if (yq[q].w & kFarFlag) continue;
        int ne = 0;
        while (ne < 2 && ((yq[q].w >> (6 * ne)) & 63)) ++ne;
        if (ne >= T.gm) continue;
        int safe = -1;
        if (T.count < kTile) {
          safe = T.count;  // empty lane: key -1 in every slot
        } else {
          for (int c = 0; c < T.count && safe < 0; ++c) {
            const int q2 = T.start + c;
            if (q2 == q || (yq[q2].w & kFarFlag)) continue;
            bool partner = false;
            for (int a = aoff[yidx[q]]; a < aoff[yidx[q] + 1] && !partner; ++a)
              partner = pos[aidx[a]] == q2;
            if (!partner) safe = c;
          }
        }
        if (safe < 0) { yq[q].w = kFarFlag; continue; }
        for (; ne < T.gm; ++ne) yq[q].w |= (safe + 1) << (6 * ne);
      }
    }
  }
  // ---- rotation-block kernel metadata in Yq.w (bits above the shuffle
  // partner lanes): "has a dedup partner", "component split over groups",
  // the point's offset from its dedup component's first point (tile order)
  {
    const std::vector<int>& ycomp = T.ycomp;
    for (const YTile& T : yt)
      for (int q = T.start; q < T.start + T.count; ++q) {
        yq[q].w |= (aoff[yidx[q] + 1] > aoff[yidx[q]] ? kPartFlag : 0) |
                   (yfar[q] ? kSplitFlag : 0) | (std::min(15, q - ycomp[q]) << kCompOffShift);
      }
  }
  // ---- guard-band risk bitmaps: per group and axis, which fraction buckets of
  // a source's rotated coordinate can put some point of the group within the
  // guard band of a bin edge.  A pair is "near" iff frac(Yq - Pq) < 2G, i.e.
  // Pq mod 2^F lies in {a, a-1, .., a-2G+1} for a = Yq mod 2^F; the buckets
  // (2^kRiskBits per axis) of those values are marked.  A source whose three
  // buckets are unmarked is "safe" for the group: none of its pairs with the
  // group can be near, and the vote kernel skips the guard-band test for it.
  // Groups with far points (every candidate exact) are never safe (flag in
  // YTile.pad[0]).
  // (only for small reference clouds: the bitmaps, 384 B per group, are read
  // per (group, unit) and must stay L1-resident; with many groups and few
  // survivors per unit -- c4 -- the lookups cost more than they save)
  const bool risk_on = R->risk_on = F >= kRiskBits + 2 && yt.size() <= 128;
  std::vector<unsigned>& risk = R->risk;
  if (risk_on) {
    const int sh = F - kRiskBits;
    const unsigned fm = (unsigned)((1u << F) - 1u);
    risk.assign(yt.size() * kRiskWords, 0u);
    for (size_t t = 0; t < yt.size(); ++t) {
      YTile& T = yt[t];
      T.pad[0] = 0;
      unsigned* bm = risk.data() + t * kRiskWords;
      for (int q = T.start; q < T.start + T.count; ++q) {
        if (yq[q].w & kFarFlag) T.pad[0] = 1;
        const int v[3] = {yq[q].x, yq[q].y, yq[q].z};
        for (int k = 0; k < 3; ++k) {
          const unsigned a = (unsigned)v[k] & fm;
          for (unsigned d : {0u, 2u * kGuard - 1u}) {  // the window [a - 2G + 1, a] spans <= 2 buckets
            const unsigned b = ((a - d) & fm) >> sh;
            bm[k * (kRiskWords / 3) + (b >> 5)] |= 1u << (b & 31);
          }
        }
      }
    }
  } else {
    risk.assign(kRiskWords, 0u);
    for (YTile& T : yt) T.pad[0] = 1;  // exact mode / few fraction bits: no source is safe
  }
  yq.push_back(make_int4(kNoRef, 0, 0, 0));  // the block kernel's empty sentinel slot (j = m_pad)
  return DSES_OK;
}

static int ref_fixed(const RefTopo& T, double inv_bin, int F, const int64_t ilo[3],
                     std::shared_ptr<const RefFixed>* out) {
  {
    std::lock_guard<std::mutex> lk(T.fmu);
    for (size_t k = T.fixed.size(); k-- > 0;) {
      const auto& c = T.fixed[k];
      if (c->F == F && c->ilo[0] == ilo[0] && c->ilo[1] == ilo[1] && c->ilo[2] == ilo[2]) {
        *out = c;
        return DSES_OK;
      }
    }
  }
  auto R = std::make_shared<RefFixed>();
  const int rc = build_ref_fixed(T, inv_bin, F, ilo, R.get());
  if (rc != DSES_OK) return rc;
  std::lock_guard<std::mutex> lk(T.fmu);
  T.fixed.push_back(R);
  if (T.fixed.size() > 4) T.fixed.erase(T.fixed.begin());
  *out = R;
  return DSES_OK;
}

// Block shape: all three sides >= 1 with at most kMaxBlockRot rotations, or
// all zero (the per-rotation kernel).
static int set_block_shape(dses_plan* P, const int* sh) {
  const bool off = sh[0] == 0 && sh[1] == 0 && sh[2] == 0;
  if (!off && (sh[0] < 1 || sh[1] < 1 || sh[2] < 1 || (int64_t)sh[0] * sh[1] * sh[2] > kMaxBlockRot))
    return fail(DSES_E_INVALID, "block shape must be 0,0,0 or three sides >= 1 with at most %d rotations",
                kMaxBlockRot);
  for (int k = 0; k < 3; ++k) P->blk_s[k] = sh[k];
  return DSES_OK;
}

int build_plan(dses_plan* P, const double* x, const double* y) {
  const int64_t n = P->n, m = P->m;
  cudaStream_t st = upload_stream(P->device);
  // ---- reference topology (cached per reference cloud and bin size)
  const std::shared_ptr<const RefTopo> topo = ref_topo(y, m, P->bin);
  // ---- fixed-point scale
  trace("fixed-point scale");
  const double ymax = topo->ymax;
  double xnorm = 0;
  for (int64_t i = 0; i < n; ++i)
    xnorm = std::max(xnorm, std::sqrt(x[3 * i] * x[3 * i] + x[3 * i + 1] * x[3 * i + 1] +
                                      x[3 * i + 2] * x[3 * i + 2]));
  double lomax = 0;
  for (int k = 0; k < 3; ++k)
    lomax = std::max(lomax, std::max(std::fabs((double)P->ilo[k]),
                                     std::fabs((double)(P->ilo[k] + P->dims[k]))));
  const double A = ymax * P->inv_bin + 3.0 * xnorm * P->inv_bin + lomax + 8.0;
  int F = 0;
  if (std::isfinite(A) && A > 0) F = (int)std::floor(std::log2(std::ldexp(1.0, 29) / A));
  F = std::min(F, 20);
  if (F < 6) F = 0;  // exact mode: every pair re-binned in binary64
  P->F = F;
  const double S = std::ldexp(1.0, F);
  const int64_t Si = (int64_t)1 << F;
  P->by = ymax;
  double tmax = 0;
  for (int k = 0; k < 3; ++k)
    tmax = std::max(tmax, (std::fabs((double)P->ilo[k]) + (double)P->dims[k]) * P->bin);
  P->bx = xnorm + tmax;

  // ---- spatial tiles
  trace("spatial tiles");
  std::vector<int> px(n);
  std::iota(px.begin(), px.end(), 0);
  std::vector<std::pair<int, int>> tx;
  kd_tiles(x, 0, n, px, tx, kTile, host_threads() >= 4 ? 2 : 0);  // source units
  std::vector<double> xs(3 * n);
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) xs[3 * i + k] = x[3 * px[i] + k];
  const double inv_s = P->inv_bin * S;
  // (the vote kernel bounds each unit by the exact box of its rotated
  // fixed-point points, computed on the device per rotation)
  std::vector<XTile> xt(tx.size());
  for (size_t t = 0; t < tx.size(); ++t) {
    XTile& T = xt[t];
    T = XTile{};
    T.start = tx[t].first;
    T.count = tx[t].second;
  }
  for (int k = 0; k < 3; ++k) { P->gorg[k] = topo->gorg[k]; P->gdim[k] = topo->gdim[k]; }
  P->gh = topo->gh;
  P->g_pts_per_cell = topo->gppc;
  P->m_pad = (int64_t)topo->yidx.size();  // reference entries (tile order)
  // fixed-point reference (cached per reference cloud, F and window origin)
  trace("fixed-point reference");
  std::shared_ptr<const RefFixed> fx;
  CK_STATUS(ref_fixed(*topo, P->inv_bin, F, P->ilo, &fx));
  const std::vector<YTile>& yt = fx->yt;
  const bool risk_on = fx->risk_on;
  if (yt.size() >= 65536 || xt.size() >= 65536)  // (group << 16 | unit) work-unit encoding
    return fail(DSES_E_LIMIT, "cloud too large for the vote kernel: at most 65535 groups / units "
                "of 32 points (about 2 million points) per cloud");
  P->near_pairs = (int64_t)topo->near.size();
  std::vector<double> xv(x, x + 3 * n);
  // ---- uploads
  // the reference cloud's arrays: uploaded once per device, then borrowed
  P->topo = topo;
  {
    std::lock_guard<std::mutex> lk(topo->dmu);
    std::shared_ptr<DeviceRef>& d = topo->dev[P->device];
    if (!d) {
      auto nd = std::make_shared<DeviceRef>();
      nd->device = P->device;
      UploadPack rp;
      static const std::vector<int> kOneZero(1, 0);
      rp.add(nd->yorig, topo->y);
      rp.add(nd->ys, topo->ys);
      rp.add(nd->near_off, topo->noff);
      rp.add(nd->near_idx, topo->nidx.empty() ? kOneZero : topo->nidx);
      rp.add(nd->ys0, topo->c0);
      rp.add(nd->ys1, topo->c1);
      rp.add(nd->ys2, topo->c2);
      rp.add(nd->ysf, topo->yf);
      rp.add(nd->gcell, topo->range);
      rp.add(nd->gpts, topo->gp);
      CK(rp.commit(nd->arena, st));
      CK(cudaStreamSynchronize(st));  // the staging buffer is reused below
      d = nd;
    }
    P->dref = d;
  }
  {
    const DeviceRef& d = *P->dref;
    P->yorig.borrow(d.yorig.p, d.yorig.cap);
    P->ys.borrow(d.ys.p, d.ys.cap);
    P->near_off.borrow(d.near_off.p, d.near_off.cap);
    P->near_idx.borrow(d.near_idx.p, d.near_idx.cap);
    P->ys0.borrow(d.ys0.p, d.ys0.cap);
    P->ys1.borrow(d.ys1.p, d.ys1.cap);
    P->ys2.borrow(d.ys2.p, d.ys2.cap);
    P->ysf.borrow(d.ysf.p, d.ysf.cap);
    P->gcell.borrow(d.gcell.p, d.gcell.cap);
    P->gpts.borrow(d.gpts.p, d.gpts.cap);
  }
  {  // the fixed-point reference layout: uploaded once per device, then borrowed
    std::lock_guard<std::mutex> lk(fx->dmu);
    std::shared_ptr<DeviceFixed>& d = fx->dev[P->device];
    if (!d) {
      auto nd = std::make_shared<DeviceFixed>();
      nd->device = P->device;
      UploadPack rp;
      rp.add(nd->yq, fx->yq);
      rp.add(nd->yt, fx->yt);
      rp.add(nd->risk, fx->risk);
      CK(rp.commit(nd->arena, st));
      CK(cudaStreamSynchronize(st));  // the staging buffer is reused below
      d = nd;
    }
    P->dfix = d;
    P->yq.borrow(d->yq.p, d->yq.cap);
    P->yt.borrow(d->yt.p, d->yt.cap);
    P->risk.borrow(d->risk.p, d->risk.cap);
  }
  // the plan's own (source- and window-dependent) arrays
  UploadPack pack;
  pack.add(P->xs, xs);
  pack.add(P->xt, xt);
  pack.add(P->x0, xv);
  CK(pack.commit(P->arena, st));
  CK(P->stats.ensure(4 * sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(P->stats.p, 0, 4 * sizeof(unsigned long long), st));
  CK(P->scal.ensure(128, st));  // [0..5] search counters, [6] sparse, [8..10] shard locals
  CK(cudaStreamSynchronize(st));  // this thread's upload stream only

  // ---- vote kernel parameters
  trace("vote kernel parameters");
  VoteParams& v = P->vp;
  v.d0 = (int)P->dims[0]; v.d1 = (int)P->dims[1]; v.d2 = (int)P->dims[2];
  if (P->sparse) return DSES_OK;  // mode queries use the sort-based path only
  v.nbins = v.d0 * v.d1 * v.d2;
  v.F = F;
  v.fmask = F ? (unsigned)(Si - 1) : 0u;
  v.D0 = (unsigned)(P->dims[0] * Si); v.D1 = (unsigned)(P->dims[1] * Si); v.D2 = (unsigned)(P->dims[2] * Si);
  v.W0 = v.D0 + 2 * kGuard; v.W1 = v.D1 + 2 * kGuard; v.W2 = v.D2 + 2 * kGuard;
  if (!F) { v.W0 = v.W1 = v.W2 = 0x7fffffffu; }  // every pair (not the sentinels) is a candidate
  else if (std::max(v.W0, std::max(v.W1, v.W2)) >= (1u << 30))
    return fail(DSES_E_INVALID, "internal: fixed-point window overflow (F=%d)", F);
  v.inv_bin = P->inv_bin;
  v.inv_s = inv_s;
  v.flo0 = (double)P->ilo[0]; v.flo1 = (double)P->ilo[1]; v.flo2 = (double)P->ilo[2];
  v.fd0 = (double)P->dims[0]; v.fd1 = (double)P->dims[1]; v.fd2 = (double)P->dims[2];
  v.n = (int)n; v.m = (int)m; v.m_pad = (int)P->m_pad;
  v.nxt = (int)xt.size(); v.nyt = (int)yt.size();
  v.xs = P->xs.as<double>(); v.ys = P->ys.as<double>(); v.yq = P->yq.as<int4>();
  v.near_off = P->near_off.as<int>(); v.near_idx = P->near_idx.as<int>();
  v.xt = P->xt.as<XTile>(); v.yt = P->yt.as<YTile>();
  v.risk = P->risk.as<unsigned>();
  v.risk_shift = risk_on ? F - kRiskBits : 0;
  v.gthr = F ? 2u * kGuard : 0xffffffffu;
  v.stats = P->stats.as<unsigned long long>();
  v.redo = nullptr;
  v.redo_n = nullptr;
  v.blk_s[0] = v.blk_s[1] = v.blk_s[2] = 0;
  {  // rotation-block kernel: list entry encoding i << jbits | j (0: no blocks)
    int jb = 1;
    while (jb < 31 && ((int64_t)1 << jb) <= P->m_pad) ++jb;  // j <= m_pad (sentinel)
    v.jbits = (((uint64_t)std::max<int64_t>(n - 1, 0) << (jb + 4)) >> 32) == 0 ? jb : 0;  // (+ 4 offset bits)
    v.ishift = v.jbits + 4;
    // DSES_BLOCK_SHAPE="a,b,c" overrides the default block shape ("0,0,0": off)
    static const std::array<int, 3> env_shape = [] {
      std::array<int, 3> v{-1, -1, -1};
      const char* e = getenv("DSES_BLOCK_SHAPE");
      if (e && *e && sscanf(e, "%d,%d,%d", &v[0], &v[1], &v[2]) != 3) v = {-1, -1, -1};
      return v;
    }();
    // Rotation blocks pay off when a source point's window holds few of a
    // reference group's points: the per-rotation kernel then idles most lanes
    // of its (source, group) steps.  Estimated lane use (identity rotation,
    // up to 32 sampled sources): reference points in the window over 32 x the
    // groups whose box meets it.  Measured (tools/block_crossover.py): c4
    // (0.07) 3.5x faster with blocks, c2 at k_trans 2-10 (0.006-0.15)
    // 2.5-1.5x, c4 at k_trans 8 (0.17) even, c2 (0.40) 0.77x.
    const double blo[3] = {((double)P->ilo[0] - 0.5) * P->bin, ((double)P->ilo[1] - 0.5) * P->bin,
                           ((double)P->ilo[2] - 0.5) * P->bin};
    const double bhi[3] = {blo[0] + (double)P->dims[0] * P->bin, blo[1] + (double)P->dims[1] * P->bin,
                           blo[2] + (double)P->dims[2] * P->bin};
    const std::vector<GroupSpan>& gs = topo->groups;
    int64_t nw = 0, gw = 0;
    const int64_t ns = std::min<int64_t>(n, 32);
    for (int64_t k = 0; k < ns; ++k) {
      const double* xi = x + 3 * (k * n / std::max<int64_t>(ns, 1));
      double wl[3], wh[3];
      for (int a = 0; a < 3; ++a) { wl[a] = xi[a] + blo[a]; wh[a] = xi[a] + bhi[a]; }
      for (size_t g = 0; g < gs.size(); ++g) {
        const double* b = &topo->gbox[6 * g];
        if (!(b[3] >= wl[0] && b[0] < wh[0] && b[4] >= wl[1] && b[1] < wh[1] && b[5] >= wl[2] && b[2] < wh[2]))
          continue;
        ++gw;
        for (int q = gs[g].start; q < gs[g].start + gs[g].count; ++q) {
          const double* yq = &topo->ys[3 * q];
          nw += (yq[0] >= wl[0]) & (yq[0] < wh[0]) & (yq[1] >= wl[1]) & (yq[1] < wh[1]) & (yq[2] >= wl[2]) &
                (yq[2] < wh[2]);
        }
      }
    }
    P->lane_use = (double)nw / (32.0 * (double)std::max<int64_t>(gw, 1));
    const bool small = P->lane_use < kBlockLaneUseMax;
    for (int k = 0; k < 3; ++k) P->blk_s[k] = small ? kDefaultBlockShape[k] : 0;
    if (env_shape[0] >= 0 && set_block_shape(P, env_shape.data()) != DSES_OK) {
      for (int k = 0; k < 3; ++k) P->blk_s[k] = 0;
    }
  }
  v.count16 = n < 65536 ? 1 : 0;
  const int64_t words = v.count16 ? (v.nbins + 1) / 2 : v.nbins;
  v.hist_words = (int)((words + 3) / 4 * 4);
  v.n_pad = (int)((n + 3) / 4 * 4);
  // shared-memory placement
  trace("shared-memory placement");
  v.unit_cap = kUnitCapMin;
  const size_t fixed = vote_smem_bytes(v, false, false, P->vote_threads);
  const size_t hb = (size_t)v.hist_words * 4, pb = (size_t)v.n_pad * 16;
  static const size_t static_smem = (vote_static_smem() + 127) & ~size_t(127);
  const size_t lim = P->smem_optin - std::max<size_t>(static_smem, 256);  // minus the kernel's static shared memory
  P->hsmem = v.count16 && fixed + hb <= lim;
  if (!P->hsmem) {  // global-memory histograms always use 32-bit counts
    v.count16 = 0;
    v.hist_words = (int)((v.nbins + 3) / 4 * 4);
  }
  P->psmem = fixed + pb + (P->hsmem ? hb : 0) <= lim;
  if (!P->hsmem && !P->psmem && fixed + pb <= lim) P->psmem = true;
  {  // spend the remaining shared memory on the (group, unit) list: fewer rounds
    const size_t used = fixed + (P->hsmem ? hb : 0) + (P->psmem ? pb : 0);
    const int64_t all = (int64_t)v.nxt * v.nyt;
    const int64_t extra = used < lim ? (int64_t)((lim - used) / 4) : 0;
    v.unit_cap = (int)std::max<int64_t>(kUnitCapMin, std::min<int64_t>(kUnitCapMin + extra,
                                                                    std::max<int64_t>(all, kUnitCapMin)));
    // a round of one group must fit all its units plus its chunk mask
    v.unit_cap = (int)std::max<int64_t>(v.unit_cap, (int64_t)v.nxt + 2);
  }
  trace("occupancy");
  int per_sm = vote_max_ctas_per_sm(v, P->hsmem, P->psmem, P->vote_threads);
  if (per_sm < 1) {
    P->vote_threads = 512;
    per_sm = vote_max_ctas_per_sm(v, P->hsmem, P->psmem, P->vote_threads);
  }
  if (per_sm < 1)
    return fail(DSES_E_LIMIT, "source cloud too large for the vote kernel: its unit boxes need "
                "%zu bytes of shared memory (about 180,000 source points at most)",
                vote_smem_bytes(v, P->hsmem, P->psmem, P->vote_threads));
  P->vote_grid = per_sm * P->sms;
  trace("plan ready");
  return DSES_OK;
}

int set_grid(dses_plan* P, const dses_grid* g, RotSource* rs, cudaStream_t st) {
  std::memset(rs, 0, sizeof(*rs));
  if (!g || g->k < 0 || !g->cos_tab || !g->sin_tab) return fail(DSES_E_INVALID, "bad rotation grid");
  const size_t nt = (size_t)(2 * g->k + 1);
  CK(P->cth.ensure(nt * 8, st));
  CK(P->sth.ensure(nt * 8, st));
  CK(h2d(P->cth.p, g->cos_tab, nt * 8, st));
  CK(h2d(P->sth.p, g->sin_tab, nt * 8, st));
  rs->cth = P->cth.as<double>();
  rs->sth = P->sth.as<double>();
  rs->rots = nullptr;
  rs->k = g->k;
  rs->has_center = g->center ? 1 : 0;
  if (g->center) std::memcpy(rs->center, g->center, sizeof(rs->center));
  return DSES_OK;
}

// Flat bins of the lattice fit the search's int32 candidate arrays.
static bool lattice_fits_int32(const dses_plan* P) {
  return (double)P->dims[0] * (double)P->dims[1] * (double)P->dims[2] < 2147483647.0;
}

static SparseParams sparse_params(const dses_plan* P, const RotSource& rs) {
  SparseParams sp{};
  sp.n = (int)P->n;
  sp.m = (int)P->m;
  sp.x = P->x0.as<double>();
  sp.y = P->yorig.as<double>();
  sp.inv_bin = P->inv_bin;
  sp.flo0 = (double)P->ilo[0]; sp.flo1 = (double)P->ilo[1]; sp.flo2 = (double)P->ilo[2];
  sp.fd0 = (double)P->dims[0]; sp.fd1 = (double)P->dims[1]; sp.fd2 = (double)P->dims[2];
  sp.d1 = P->dims[1];
  sp.d2 = P->dims[2];
  sp.rot = rs;
  return sp;
}

// Sort-based mode batch (the reference's mode_sparse_batch, _kernels.py:196-294)
// for lattices beyond kDenseMaxBins.  When the lattice has < 2^31 bins the
// flat bins are also narrowed to the int32 array the search's select / score
// stages read, so dses() runs on such lattices like the reference
// (mode_search.py:158-163 dispatches them to its sparse kernel).
int run_sparse(dses_plan* P, const RotSource& rs, int64_t r_begin, int64_t r_count, cudaStream_t st) {
  CK(P->counts.ensure(sizeof(int) * std::max<int64_t>(r_count, 1), st));
  CK(P->lins64.ensure(sizeof(long long) * std::max<int64_t>(r_count, 1), st));
  CK(P->ties.ensure(sizeof(int) * std::max<int64_t>(r_count, 1), st));
  P->cur_r_begin = r_begin;
  P->cur_r_count = r_count;
  P->cur_rot = rs;
  if (r_count <= 0) return DSES_OK;
  const SparseParams sp = sparse_params(P, rs);
  const size_t sb = sparse_scratch_bytes(P->n, P->m);
  CK(P->sparse_scratch.ensure(sb, st));
  CK(P->scal.ensure(64, st));
  CK(launched(launch_sparse_modes(sp, r_begin, r_count, P->sparse_scratch.p, P->sparse_scratch.cap,
                                  P->scal.as<unsigned long long>() + 6, P->counts.as<int>(),
                                  P->lins64.as<long long>(), P->ties.as<int>(), P->sms, st),
              (int)(5 * r_count)));
  if (lattice_fits_int32(P)) {
    CK(P->lins.ensure(sizeof(int) * std::max<int64_t>(r_count, 1), st));
    CK(launched(launch_narrow_lins(P->lins64.as<long long>(), P->lins.as<int>(), r_count, P->sms, st)));
  }
  return DSES_OK;
}

// Rotation-block kernel eligibility: grid rotations (blocks are boxes of the
// grid), shared-memory histogram and points, fixed-point binning, and the
// entry word i << (jbits + 4) | j << 4 | c in 32 bits (n * m_pad < 2^28).
static bool blocks_enabled(const dses_plan* P) {
  return P->blk_s[0] > 0 && P->hsmem && P->psmem && P->F > 0 && P->vp.jbits > 0 && !P->sparse;
}
static bool use_blocks(const dses_plan* P, const RotSource& rs) {
  return blocks_enabled(P) && rs.cth && !rs.rots;
}

int run_vote(dses_plan* P, const RotSource& rs, int64_t r_begin, int64_t r_count, cudaStream_t st) {
  if (P->sparse) return run_sparse(P, rs, r_begin, r_count, st);
  CK(P->counts.ensure(sizeof(int) * std::max<int64_t>(r_count, 1), st));
  CK(P->lins.ensure(sizeof(int) * std::max<int64_t>(r_count, 1), st));
  CK(P->ties.ensure(sizeof(int) * std::max<int64_t>(r_count, 1), st));
  VoteParams v = P->vp;
  v.rot = rs;
  v.r_begin = r_begin;
  v.r_count = r_count;
  v.counts = P->counts.as<int>();
  v.lins = P->lins.as<int>();
  v.ties = P->ties.as<int>();
  P->cur_r_begin = r_begin;
  P->cur_r_count = r_count;
  P->cur_rot = rs;
  if (r_count <= 0) return DSES_OK;
  int grid = (int)std::min<int64_t>(P->vote_grid_cap > 0 ? P->vote_grid_cap : P->vote_grid, r_count);
  // global-memory fallbacks: one slab per CTA, at most ~4 GiB in total
  const size_t per_cta = (P->hsmem ? 0 : (size_t)v.hist_words * 4) + (P->psmem ? 0 : (size_t)v.n_pad * 16);
  if (per_cta) {
    const size_t budget = (size_t)4 << 30;
    grid = (int)std::max<size_t>(1, std::min<size_t>((size_t)grid, budget / per_cta));
    if (!P->hsmem) {
      CK(P->hist_g.ensure((size_t)grid * v.hist_words * 4, st));
      v.hist_global = P->hist_g.as<unsigned>();
    }
    if (!P->psmem) {
      CK(P->p_g.ensure((size_t)grid * v.n_pad * 16, st));
      v.p_global = P->p_g.as<int4>();
    }
  }
  CK(cudaEventRecord(P->ev[5], st));
  CK(cudaMemsetAsync(v.stats + 3, 0, sizeof(unsigned long long), st));  // rotation queue
  if (use_blocks(P, rs)) {
    // rotation blocks: one candidate list per box of neighbouring rotations; blocks
    // whose list overflows the slab are re-run by the per-rotation kernel
    for (int k = 0; k < 3; ++k) v.blk_s[k] = P->blk_s[k];
    v.list_cap = P->blk_cap;
    CK(P->blist.ensure(((size_t)grid * v.list_cap + kBlockListSlack) * 16, st, false));  // 16-byte entries
    CK(P->redo.ensure(8 * (size_t)(r_count + 1), st));
    v.list = P->blist.as<unsigned>();
    v.redo_n = P->redo.as<unsigned long long>();
    v.redo = P->redo.as<long long>() + 1;
    CK(cudaMemsetAsync(v.redo_n, 0, 8, st));
    CK(launched(launch_vote_blocks(v, grid, P->vote_threads, st)));
    CK(cudaMemsetAsync(v.stats + 3, 0, sizeof(unsigned long long), st));
    CK(launched(launch_vote_redo(v, grid, P->vote_threads, st)));
  } else {
    CK(launched(launch_vote(v, P->hsmem, P->psmem, grid, P->vote_threads, st)));
  }
  CK(cudaEventRecord(P->ev[6], st));
  P->vote_timed = true;
  return DSES_OK;
}

ScoreParams score_params(const dses_plan* P, const RotSource& rs, int code, double param) {
  ScoreParams s{};
  s.n = (int)P->n;
  s.m = (int)P->m;
  s.x = P->x0.as<double>();
  s.ys0 = P->ys0.as<double>();
  s.ys1 = P->ys1.as<double>();
  s.ys2 = P->ys2.as<double>();
  s.ysf = P->ysf.as<float4>();
  s.rot = rs;
  s.bin_size = P->bin;
  s.ilo0 = P->ilo[0]; s.ilo1 = P->ilo[1]; s.ilo2 = P->ilo[2];
  s.d1 = (int)P->dims[1]; s.d2 = (int)P->dims[2];
  s.code = code;
  s.param = param;
  s.paramf = (float)param;
  s.halff = (float)(0.5 * param);
  // per-axis |d32 - d64| <= 2^-24 (|y| + |p| + |d|) <= 2^-23 (bx + by); margin x2
  s.amb = (float)(2.0 * std::ldexp(P->bx + P->by, -23));
  s.tvec = nullptr;
  s.exh_k = -1;
  s.gcell = P->gcell.as<int2>();
  s.gpts = P->gpts.as<float4>();
  for (int k = 0; k < 3; ++k) { s.gorg[k] = P->gorg[k]; s.gdim[k] = P->gdim[k]; }
  s.gh = P->gh;
  s.ginv = 1.0f / P->gh;
  s.gppc = P->g_pts_per_cell;
  return s;
}

// rigorous bound on |screen - exact| per candidate
double screen_tolerance(const dses_plan* P, int code) {
  if (code == kSatL0) return 0.0;
  const double e_pt = 8.0 * std::ldexp(P->bx + P->by, -23);
  return 2.0 * (double)P->n * e_pt;
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" int dses_plan_create(int device, const double* x, int64_t n, const double* y, int64_t m,
                                double bin_size, const int64_t ilo[3], const int64_t dims[3],
                                dses_plan** out) {
  if (!out) return fail(DSES_E_INVALID, "out is NULL");
  *out = nullptr;
  if (!x || !y || n < 1 || m < 1) return fail(DSES_E_INVALID, "empty cloud");
  if (n >= (1ll << 31) || m >= (1ll << 30)) return fail(DSES_E_INVALID, "cloud too large");
  if (!(bin_size > 0) || !std::isfinite(bin_size)) return fail(DSES_E_INVALID, "bad bin size");
  for (int k = 0; k < 3; ++k)
    if (dims[k] < 1) return fail(DSES_E_INVALID, "dims must be positive");
  const double nbins = (double)dims[0] * (double)dims[1] * (double)dims[2];
  if (nbins * (double)n >= 4.611686018427388e18)  // the reference's key-space guard (mode_search.py:149-152)
    return fail(DSES_E_INVALID, "translation lattice too large");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(DSES_E_NODEVICE, "no CUDA device");
  if (device < 0 || device >= ndev) return fail(DSES_E_INVALID, "bad device %d", device);
  trace("set device");
  CK(cudaSetDevice(device));
  keep_pool(device);
  // individual attributes: cudaGetDeviceProperties costs up to tens of ms per call
  int major = 0, minor = 0, sms = 0, optin = 0;
  CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  CK(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  if (major != 10) return fail(DSES_E_NODEVICE, "sm_100a build cannot run on sm_%d%d", major, minor);
  dses_plan* P = new dses_plan();
  P->device = device;
  P->sms = sms;
  P->smem_optin = (size_t)optin;
  P->n = n;
  P->m = m;
  P->bin = bin_size;
  P->inv_bin = 1.0 / bin_size;  // mode_search.py:157 (inv_bin = 1.0 / bin_size)
  for (int k = 0; k < 3; ++k) { P->ilo[k] = ilo[k]; P->dims[k] = dims[k]; }
  P->sparse = nbins > (double)kDenseMaxBins;
  for (auto& e : P->ev) cudaEventCreate(&e);
  P->rec_host = rec_take();
  if (!P->rec_host) { dses_plan_destroy(P); return fail(DSES_E_NOMEM, "pinned record"); }
  TrafficScope ts_(P);
  int rc;
  try {  // no C++ exception may cross the C ABI (host allocations of the layout)
    rc = build_plan(P, x, y);
  } catch (const std::bad_alloc&) {
    rc = fail(DSES_E_NOMEM, "host memory exhausted building the plan");
  } catch (const std::exception& e) {
    rc = fail(DSES_E_CUDA, "plan construction failed: %s", e.what());
  }
  if (rc != DSES_OK) { dses_plan_destroy(P); return rc; }
  *out = P;
  return DSES_OK;
}

extern "C" int dses_plan_destroy(dses_plan* P) {
  if (!P) return DSES_OK;
  cudaSetDevice(P->device);
  DevBuf* bufs[] = {&P->risk, &P->xs, &P->ys, &P->yq, &P->near_off, &P->near_idx, &P->xt, &P->yt,
                    &P->x0, &P->ys0, &P->ys1, &P->ys2, &P->ysf, &P->gcell, &P->gpts, &P->arena, &P->yorig, &P->lins64, &P->sparse_scratch, &P->cth, &P->sth, &P->rots,
                    &P->counts, &P->lins, &P->ties, &P->hist_g, &P->p_g, &P->stats, &P->scal,
                    &P->cand_rows, &P->cand_lins, &P->err32, &P->partial, &P->sel, &P->vals,
                    &P->err64, &P->win_err, &P->win_row, &P->win_c, &P->tmp_rows, &P->tmp_lins,
                    &P->tvec, &P->blist, &P->redo};
  if (P->pend.active) cudaEventSynchronize(P->ev[4]);  // an unwaited search
  for (DevBuf* b : bufs) b->release();
  for (auto& e : P->ev) cudaEventDestroy(e);
  rec_give(P->rec_host);
  delete P;
  return DSES_OK;
}

extern "C" int dses_plan_info(const dses_plan* P, int64_t* frac_bits, int64_t* x_tiles,
                              int64_t* y_tiles, int64_t* near_pairs) {
  if (!P) return fail(DSES_E_INVALID, "null plan");
  if (frac_bits) *frac_bits = P->F;
  if (x_tiles) *x_tiles = P->vp.nxt;
  if (y_tiles) *y_tiles = P->vp.nyt;
  if (near_pairs) *near_pairs = P->near_pairs;
  return DSES_OK;
}

extern "C" int dses_plan_set_vote_grid(dses_plan* P, int64_t ctas) {
  if (!P) return fail(DSES_E_INVALID, "null plan");
  if (ctas < 0) return fail(DSES_E_INVALID, "negative CTA count");
  P->vote_grid_cap = (int)std::min<int64_t>(ctas, P->vote_grid);
  return DSES_OK;
}

extern "C" int dses_plan_blocks(const dses_plan* P, int64_t* shape) {
  if (!P || !shape) return fail(DSES_E_INVALID, "null argument");
  for (int k = 0; k < 3; ++k) shape[k] = blocks_enabled(P) ? P->blk_s[k] : 0;
  return DSES_OK;
}

extern "C" int dses_plan_set_blocks(dses_plan* P, const int64_t* shape, int64_t list_cap) {
  if (!P || !shape) return fail(DSES_E_INVALID, "null argument");
  if (list_cap < 0 || list_cap > kBlockListCap) return fail(DSES_E_INVALID, "list capacity must be in [0, %d]", kBlockListCap);
  const int sh[3] = {(int)std::max<int64_t>(std::min<int64_t>(shape[0], 1 << 20), -1),
                     (int)std::max<int64_t>(std::min<int64_t>(shape[1], 1 << 20), -1),
                     (int)std::max<int64_t>(std::min<int64_t>(shape[2], 1 << 20), -1)};
  CK_STATUS(set_block_shape(P, sh));
  P->blk_cap = list_cap > 0 ? (int)((list_cap + 31) / 32 * 32) : kBlockListCap;
  return DSES_OK;
}

static int fetch_modes(dses_plan* P, int64_t nrot, int64_t* counts, int64_t* lins, int64_t* ties,
                       cudaStream_t st) {
  std::vector<int> c(nrot), l(nrot), t(nrot);
  std::vector<long long> l64(P->sparse ? nrot : 0);
  if (nrot > 0) {
    CK(d2h(c.data(), P->counts.p, 4 * nrot, st));
    if (P->sparse) CK(d2h(l64.data(), P->lins64.p, 8 * nrot, st));
    else CK(d2h(l.data(), P->lins.p, 4 * nrot, st));
    CK(d2h(t.data(), P->ties.p, 4 * nrot, st));
  }
  CK(cudaStreamSynchronize(st));
  for (int64_t r = 0; r < nrot; ++r) {
    if (counts) counts[r] = c[r];
    if (lins) lins[r] = P->sparse ? (int64_t)l64[r] : (int64_t)l[r];
    if (ties) ties[r] = t[r];
  }
  return DSES_OK;
}

extern "C" int dses_mode_batch(dses_plan* P, const double* rots, int64_t nrot, int64_t* counts,
                               int64_t* lins, int64_t* ties, void* stream) {
  TrafficScope ts_(P);
  if (!P || (!rots && nrot > 0) || nrot < 0) return fail(DSES_E_INVALID, "bad arguments");
  CK(cudaSetDevice(P->device));
  cudaStream_t st = (cudaStream_t)stream;
  CK(P->rots.ensure(sizeof(double) * 9 * std::max<int64_t>(nrot, 1), st));
  if (nrot > 0) CK(h2d(P->rots.p, rots, sizeof(double) * 9 * nrot, st));
  RotSource rs{};
  rs.rots = P->rots.as<double>();
  int rc = run_vote(P, rs, 0, nrot, st);
  if (rc) return rc;
  return fetch_modes(P, nrot, counts, lins, ties, st);
}

extern "C" int dses_mode_grid(dses_plan* P, const dses_grid* g, int64_t r_begin, int64_t nrot,
                              int64_t* counts, int64_t* lins, int64_t* ties, void* stream) {
  TrafficScope ts_(P);
  if (!P || nrot < 0 || r_begin < 0) return fail(DSES_E_INVALID, "bad arguments");
  CK(cudaSetDevice(P->device));
  cudaStream_t st = (cudaStream_t)stream;
  RotSource rs;
  int rc = set_grid(P, g, &rs, st);
  if (rc) return rc;
  const int64_t total = (2 * g->k + 1) * (2 * g->k + 1) * (2 * g->k + 1);
  if (r_begin + nrot > total) return fail(DSES_E_INVALID, "rotation range beyond the grid");
  rc = run_vote(P, rs, r_begin, nrot, st);
  if (rc) return rc;
  return fetch_modes(P, nrot, counts, lins, ties, st);
}

extern "C" int dses_mode_dense_batch(int device, const double* rots, int64_t nrot, const double* x,
                                     int64_t n, const double* y, int64_t m, double bin_size,
                                     const int64_t ilo[3], const int64_t dims[3], int64_t* counts,
                                     int64_t* lins, int64_t* ties) {
  dses_plan* P = nullptr;
  int rc = dses_plan_create(device, x, n, y, m, bin_size, ilo, dims, &P);
  if (rc) return rc;
  rc = dses_mode_batch(P, rots, nrot, counts, lins, ties, nullptr);
  dses_plan_destroy(P);
  return rc;
}

extern "C" int dses_translation_histogram(dses_plan* P, const double* rot, int dedup,
                                          int64_t* lins, int64_t* counts, int64_t cap,
                                          int64_t* nbins, int64_t* npairs, void* stream) {
  TrafficScope ts_(P);
  if (!P || !rot || !nbins || cap < 0 || (cap > 0 && (!lins || !counts)))
    return fail(DSES_E_INVALID, "bad arguments");
  CK(cudaSetDevice(P->device));
  cudaStream_t st = (cudaStream_t)stream;
  CK(P->rots.ensure(sizeof(double) * 9, st));
  CK(h2d(P->rots.p, rot, sizeof(double) * 9, st));
  RotSource rs{};
  rs.rots = P->rots.as<double>();
  const SparseParams sp = sparse_params(P, rs);
  CK(P->sparse_scratch.ensure(sparse_scratch_bytes(P->n, P->m), st));
  CK(P->scal.ensure(64, st));
  unsigned long long* dl = nullptr;
  int *dc = nullptr, *dn = nullptr;
  unsigned long long nk = 0;
  CK(launched(launch_sparse_histogram(sp, dedup != 0, P->sparse_scratch.p, P->sparse_scratch.cap,
                                      P->scal.as<unsigned long long>() + 6, &dl, &dc, &dn, &nk,
                                      P->sms, st),
              dedup ? 5 : 4));
  int nr = 0;
  CK(d2h(&nr, dn, sizeof nr, st));
  *nbins = nr;
  if (npairs) *npairs = (int64_t)nk;
  if (nr > cap) return fail(DSES_E_INVALID, "histogram has more bins than cap");
  std::vector<unsigned long long> hl(nr);
  std::vector<int> hc(nr);
  if (nr > 0) {
    CK(d2h(hl.data(), dl, sizeof(unsigned long long) * nr, st));
    CK(d2h(hc.data(), dc, sizeof(int) * nr, st));
  }
  for (int k = 0; k < nr; ++k) {
    lins[k] = (int64_t)hl[k];
    counts[k] = hc[k];
  }
  return DSES_OK;
}

extern "C" int dses_refine_batch(dses_plan* P, const double* rots, const double* ts, int64_t ncand,
                                 int code, double param, double* out, void* stream) {
  TrafficScope ts_(P);
  if (!P || ncand < 0 || (ncand > 0 && (!rots || !ts || !out)) || code < 0 || code > 4)
    return fail(DSES_E_INVALID, "bad arguments");
  if (ncand == 0) return DSES_OK;
  CK(cudaSetDevice(P->device));
  cudaStream_t st = (cudaStream_t)stream;
  CK(P->rots.ensure(sizeof(double) * 9 * ncand, st));
  CK(P->tvec.ensure(sizeof(double) * 3 * ncand, st));
  CK(P->tmp_rows.ensure(sizeof(int64_t) * ncand, st));
  CK(P->tmp_lins.ensure(sizeof(int) * ncand, st));
  CK(P->vals.ensure(sizeof(double) * P->n * ncand, st));
  CK(P->err64.ensure(sizeof(double) * ncand, st));
  std::vector<int64_t> rows(ncand);
  std::iota(rows.begin(), rows.end(), 0);
  std::vector<int> zeros(ncand, 0);
  CK(h2d(P->rots.p, rots, sizeof(double) * 9 * ncand, st));
  CK(h2d(P->tvec.p, ts, sizeof(double) * 3 * ncand, st));
  CK(h2d(P->tmp_rows.p, rows.data(), sizeof(int64_t) * ncand, st));
  CK(h2d(P->tmp_lins.p, zeros.data(), sizeof(int) * ncand, st));
  RotSource rs{};
  rs.rots = P->rots.as<double>();
  ScoreParams s = score_params(P, rs, code, param);
  s.tvec = P->tvec.as<double>();
  CK(launched(launch_exact(s, P->tmp_rows.as<int64_t>(), P->tmp_lins.as<int>(), nullptr, ncand,
                           P->vals.as<double>(), P->err64.as<double>(), st),
              (int)((ncand + 65534) / 65535) + 1));
  CK(d2h(out, P->err64.p, sizeof(double) * ncand, st));
  CK(cudaStreamSynchronize(st));
  return DSES_OK;
}

// ---- stages -------------------------------------------------------------
extern "C" int dses_stage_vote(dses_plan* P, const dses_grid* g, int64_t r_begin, int64_t r_count,
                               int64_t* mstar_local, int64_t* valid_local, void* stream) {
  TrafficScope ts_(P);
  if (!P || !g) return fail(DSES_E_INVALID, "bad arguments");
  if (!lattice_fits_int32(P))
    return fail(DSES_E_LIMIT, "translation window of %.3g bins: the search supports lattices "
                "below 2^31 bins (mode queries, dses_mode_*, support any size)",
                (double)P->dims[0] * P->dims[1] * P->dims[2]);
  CK(cudaSetDevice(P->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t total = (2 * g->k + 1) * (2 * g->k + 1) * (2 * g->k + 1);
  if (r_count < 0) r_count = total - r_begin;
  if (r_begin < 0 || r_begin + r_count > total) return fail(DSES_E_INVALID, "rotation range beyond the grid");
  RotSource rs;
  int rc = set_grid(P, g, &rs, st);
  if (rc) return rc;
  P->cur_k = g->k;
  rc = run_vote(P, rs, r_begin, r_count, st);
  if (rc) return rc;
  unsigned long long* sc = P->scal.as<unsigned long long>();
  CK(cudaMemsetAsync(sc, 0, 2 * sizeof(unsigned long long), st));
  if (r_count > 0) CK(launched(launch_select_stats(P->counts.as<int>(), r_count, sc, sc + 1, P->sms, st)));
  unsigned long long h[2];
  CK(d2h(h, sc, sizeof h, st));
  CK(cudaStreamSynchronize(st));
  if (mstar_local) *mstar_local = (int64_t)h[0];
  if (valid_local) *valid_local = (int64_t)h[1];
  return DSES_OK;
}

extern "C" int dses_stage_argmax(dses_plan* P, int64_t mstar_global, int64_t* row_local, void* stream) {
  TrafficScope ts_(P);
  if (!P || !row_local) return fail(DSES_E_INVALID, "bad arguments");
  CK(cudaSetDevice(P->device));
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* sc = P->scal.as<unsigned long long>() + 2;
  CK(cudaMemsetAsync(sc, 0xff, sizeof(unsigned long long), st));
  if (P->cur_r_count > 0)
    CK(launched(launch_argmax(P->counts.as<int>(), P->cur_r_count, P->cur_r_begin,
                              (int)mstar_global, sc, P->sms, st)));
  unsigned long long h;
  CK(d2h(&h, sc, sizeof h, st));
  CK(cudaStreamSynchronize(st));
  *row_local = h == ~0ull ? INT64_MAX : (int64_t)h;
  return DSES_OK;
}

extern "C" int dses_stage_screen(dses_plan* P, double q, int64_t mstar_global, int code,
                                 double param, int64_t* kept_local, double* min32_local, double* tol,
                                 void* stream) {
  TrafficScope ts_(P);
  if (!P || code < 0 || code > 4) return fail(DSES_E_INVALID, "bad arguments");
  CK(cudaSetDevice(P->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nr = P->cur_r_count;
  // engines.py:196-201 in binary64: cutoff = q * M* - 1e-9
  const double cutoff = q * (double)mstar_global - 1e-9;
  CK(P->cand_rows.ensure(sizeof(int64_t) * std::max<int64_t>(nr, 1), st));
  CK(P->cand_lins.ensure(sizeof(int) * std::max<int64_t>(nr, 1), st));
  unsigned long long* sc = P->scal.as<unsigned long long>() + 3;
  CK(cudaMemsetAsync(sc, 0, sizeof(unsigned long long), st));
  if (nr > 0)
    CK(launched(launch_compact(P->counts.as<int>(), P->lins.as<int>(), nr, P->cur_r_begin, cutoff,
                               P->cand_rows.as<int64_t>(), P->cand_lins.as<int>(), sc, P->sms, st)));
  unsigned long long kept;
  CK(d2h(&kept, sc, sizeof kept, st));
  CK(cudaStreamSynchronize(st));
  P->kept = (int64_t)kept;
  if (kept_local) *kept_local = (int64_t)kept;
  if (tol) *tol = screen_tolerance(P, code);
  if (kept == 0) {
    if (min32_local) *min32_local = INFINITY;
    return DSES_OK;
  }
  const int nblk = (int)((P->n + screen_threads() - 1) / screen_threads());
  CK(P->partial.ensure(sizeof(double) * nblk * kept, st));
  CK(P->err32.ensure(sizeof(double) * kept, st));
  unsigned long long* mb = P->scal.as<unsigned long long>() + 4;
  CK(cudaMemsetAsync(mb, 0x7f, sizeof(unsigned long long), st));
  ScoreParams s = score_params(P, P->cur_rot, code, param);
  CK(launched(launch_screen(s, P->cand_rows.as<int64_t>(), P->cand_lins.as<int>(), (int64_t)kept,
                            P->partial.as<double>(), P->err32.as<double>(), mb, st),
              (int)((kept + 65534) / 65535) + 1));
  double mn;
  CK(d2h(&mn, mb, sizeof mn, st));
  CK(cudaStreamSynchronize(st));
  if (min32_local) *min32_local = mn;
  return DSES_OK;
}

extern "C" int dses_stage_rescore(dses_plan* P, double threshold, int code, double param,
                                  double* err_local, int64_t* row_local, int64_t* rescored,
                                  void* stream) {
  TrafficScope ts_(P);
  if (!P || code < 0 || code > 4) return fail(DSES_E_INVALID, "bad arguments");
  CK(cudaSetDevice(P->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (err_local) *err_local = INFINITY;
  if (row_local) *row_local = INT64_MAX;
  if (rescored) *rescored = 0;
  if (P->kept <= 0) return DSES_OK;
  CK(P->sel.ensure(sizeof(int) * P->kept, st));
  unsigned long long* ns = P->scal.as<unsigned long long>() + 5;
  CK(cudaMemsetAsync(ns, 0, sizeof(unsigned long long), st));
  CK(launched(launch_rescore_compact(P->err32.as<double>(), P->kept, threshold, P->sel.as<int>(), ns, st)));
  unsigned long long nsel;
  CK(d2h(&nsel, ns, sizeof nsel, st));
  CK(cudaStreamSynchronize(st));
  if (rescored) *rescored = (int64_t)nsel;
  if (nsel == 0) return DSES_OK;
  CK(P->vals.ensure(sizeof(double) * P->n * nsel, st));
  CK(P->err64.ensure(sizeof(double) * nsel, st));
  CK(P->win_err.ensure(sizeof(double), st));
  CK(P->win_row.ensure(sizeof(int64_t), st));
  CK(P->win_c.ensure(sizeof(int), st));
  ScoreParams s = score_params(P, P->cur_rot, code, param);
  CK(launched(launch_exact(s, P->cand_rows.as<int64_t>(), P->cand_lins.as<int>(), P->sel.as<int>(),
                           (int64_t)nsel, P->vals.as<double>(), P->err64.as<double>(), st),
              (int)((nsel + 65534) / 65535) + 1));
  CK(launched(launch_winner(P->err64.as<double>(), P->sel.as<int>(), P->cand_rows.as<int64_t>(),
                            (int64_t)nsel, P->win_err.as<double>(), P->win_row.as<int64_t>(),
                            P->win_c.as<int>(), st)));
  double e;
  int64_t r;
  CK(d2h(&e, P->win_err.p, sizeof e, st));
  CK(d2h(&r, P->win_row.p, sizeof r, st));
  CK(cudaStreamSynchronize(st));
  if (err_local) *err_local = e;
  if (row_local) *row_local = r;
  return DSES_OK;
}

extern "C" int dses_stage_row_info(dses_plan* P, int64_t row, int64_t* lin, int64_t* count,
                                   void* stream) {
  TrafficScope ts_(P);
  if (!P) return fail(DSES_E_INVALID, "null plan");
  const int64_t rr = row - P->cur_r_begin;
  if (rr < 0 || rr >= P->cur_r_count) return fail(DSES_E_INVALID, "row %lld not in this plan's slice", (long long)row);
  CK(cudaSetDevice(P->device));
  cudaStream_t st = (cudaStream_t)stream;
  int l, c;
  CK(d2h(&l, P->lins.as<int>() + rr, 4, st));
  CK(d2h(&c, P->counts.as<int>() + rr, 4, st));
  CK(cudaStreamSynchronize(st));
  if (lin) *lin = l;
  if (count) *count = c;
  return DSES_OK;
}

extern "C" int dses_pose_error(dses_plan* P, const dses_grid* g, int64_t row, int64_t lin, int code,
                               double param, double* err, void* stream) {
  TrafficScope ts_(P);
  if (!P || !err || code < 0 || code > 4 || lin < 0) return fail(DSES_E_INVALID, "bad arguments");
  CK(cudaSetDevice(P->device));
  cudaStream_t st = (cudaStream_t)stream;
  RotSource rs;
  int rc = set_grid(P, g, &rs, st);
  if (rc) return rc;
  CK(P->tmp_rows.ensure(sizeof(int64_t), st));
  CK(P->tmp_lins.ensure(sizeof(int), st));
  CK(P->vals.ensure(sizeof(double) * P->n, st));
  CK(P->err64.ensure(sizeof(double), st));
  const int l32 = (int)lin;
  CK(h2d(P->tmp_rows.p, &row, sizeof row, st));
  CK(h2d(P->tmp_lins.p, &l32, sizeof l32, st));
  ScoreParams s = score_params(P, rs, code, param);
  CK(launched(launch_exact(s, P->tmp_rows.as<int64_t>(), P->tmp_lins.as<int>(), nullptr, 1,
                           P->vals.as<double>(), P->err64.as<double>(), st), 2));
  CK(d2h(err, P->err64.p, sizeof(double), st));
  CK(cudaStreamSynchronize(st));
  return DSES_OK;
}

extern "C" int dses_stage_stats(dses_plan* P, int64_t* pairs, int64_t* votes, int64_t* rechecks) {
  TrafficScope ts_(P);
  if (!P) return fail(DSES_E_INVALID, "null plan");
  CK(cudaSetDevice(P->device));
  unsigned long long h[3];
  CK(cudaMemcpy(h, P->stats.p, sizeof h, cudaMemcpyDeviceToHost));
  CK(cudaMemset(P->stats.p, 0, sizeof h));
  if (pairs) *pairs = (int64_t)h[0];
  if (votes) *votes = (int64_t)h[1];
  if (rechecks) *rechecks = (int64_t)h[2];
  return DSES_OK;
}

// At most this many screened candidates are re-scored inside the fused tail
// (more -- a flat landscape of near-ties -- falls back to the staged path).
static constexpr int64_t kFusedRescoreCap = 4096;

// Every device buffer a dses_search over `nr` rotations touches, allocated up
// front (plan construction via dses_plan_reserve, or at the top of the
// search): a search never grows the memory pool between its launches.
static int reserve_search(dses_plan* P, int64_t nr, cudaStream_t st = 0) {
  nr = std::max<int64_t>(nr, 1);
  CK(P->counts.ensure(sizeof(int) * nr, st));
  CK(P->lins.ensure(sizeof(int) * nr, st));
  CK(P->ties.ensure(sizeof(int) * nr, st));
  const VoteParams& v = P->vp;
  const size_t per_cta = (P->hsmem ? 0 : (size_t)v.hist_words * 4) + (P->psmem ? 0 : (size_t)v.n_pad * 16);
  if (per_cta && !P->sparse) {
    const size_t budget = (size_t)4 << 30;
    const int grid = (int)std::max<size_t>(
        1, std::min<size_t>((size_t)std::min<int64_t>(P->vote_grid, nr), budget / per_cta));
    if (!P->hsmem) CK(P->hist_g.ensure((size_t)grid * v.hist_words * 4, st));
    if (!P->psmem) CK(P->p_g.ensure((size_t)grid * v.n_pad * 16, st));
  }
  if (blocks_enabled(P)) {
    CK(P->blist.ensure(((size_t)P->vote_grid * P->blk_cap + kBlockListSlack) * 16, st, false));  // rotation-block lists
    CK(P->redo.ensure(8 * (size_t)(nr + 1), st));
  }
  const int64_t cap = std::min<int64_t>(nr, kFusedRescoreCap);
  const int nblk = (int)((P->n + screen_threads() - 1) / screen_threads());
  CK(P->cand_rows.ensure(sizeof(int64_t) * nr, st));
  CK(P->cand_lins.ensure(sizeof(int) * nr, st));
  CK(P->win_err.ensure(sizeof(double), st));
  CK(P->win_row.ensure(sizeof(int64_t), st));
  CK(P->win_c.ensure(sizeof(int), st));
  CK(P->tvec.ensure(sizeof(double) * (P->n + 16), st));
  CK(P->partial.ensure(sizeof(double) * nblk * nr, st));
  CK(P->err32.ensure(sizeof(double) * nr, st));
  CK(P->sel.ensure(sizeof(int) * nr, st));
  CK(P->vals.ensure(sizeof(double) * P->n * cap, st));
  CK(P->err64.ensure(sizeof(double) * cap, st));
  return DSES_OK;
}

extern "C" int dses_plan_reserve(dses_plan* P, int64_t r_count) {
  if (!P || r_count < 0) return fail(DSES_E_INVALID, "bad arguments");
  CK(cudaSetDevice(P->device));
  cudaStream_t st = upload_stream(P->device);
  const int rc = reserve_search(P, r_count, st);
  if (rc) return rc;
  CK(cudaStreamSynchronize(st));
  return DSES_OK;
}

extern "C" int dses_search_async(dses_plan* P, const dses_grid* g, int64_t r_begin,
                                 int64_t r_count, double q, int code, double param, int skip_refine,
                                 void* stream) {
  // engines.dses on one GPU.  After the vote, every stage reads the previous
  // stage's counters on the device (M*, kept, screened minimum, selected), so
  // the whole search is one stream of launches and ONE device->host read
  // (into the plan's pinned record); dses_search_wait completes it.
  TrafficScope ts_(P);
  if (!P || !g || code < 0 || code > 4) return fail(DSES_E_INVALID, "bad arguments");
  if (P->pend.active) return fail(DSES_E_INVALID, "plan has a search in flight");
  CK(cudaSetDevice(P->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t total = (2 * g->k + 1) * (2 * g->k + 1) * (2 * g->k + 1);
  if (r_count < 0) r_count = total - r_begin;
  if (r_begin < 0 || r_begin + r_count > total) return fail(DSES_E_INVALID, "rotation range beyond the grid");
  if (!lattice_fits_int32(P))
    return fail(DSES_E_LIMIT, "translation window of %.3g bins: the search supports lattices "
                "below 2^31 bins (mode queries, dses_mode_*, support any size)",
                (double)P->dims[0] * P->dims[1] * P->dims[2]);
  {
    const int rr = reserve_search(P, r_count);
    if (rr) return rr;
  }
  CK(cudaEventRecord(P->ev[0], st));
  RotSource rs;
  int rc = set_grid(P, g, &rs, st);
  if (rc) return rc;
  P->cur_k = g->k;
  rc = run_vote(P, rs, r_begin, r_count, st);
  if (rc) return rc;
  const int64_t nr = std::max<int64_t>(r_count, 1);
  unsigned long long* sc = P->scal.as<unsigned long long>();
  // scal: [0] M* [1] valid [2] argmax row [3] kept [4] min screen bits [5] selected
  CK(cudaMemsetAsync(sc, 0, 6 * sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(sc + 2, 0xff, sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(sc + 4, 0x7f, sizeof(unsigned long long), st));
  if (r_count > 0) CK(launched(launch_select_stats(P->counts.as<int>(), r_count, sc, sc + 1, P->sms, st)));
  CK(cudaEventRecord(P->ev[1], st));
  CK(P->cand_rows.ensure(sizeof(int64_t) * nr, st));
  CK(P->cand_lins.ensure(sizeof(int) * nr, st));
  CK(P->win_err.ensure(sizeof(double), st));
  CK(P->win_row.ensure(sizeof(int64_t), st));
  CK(P->win_c.ensure(sizeof(int), st));
  CK(P->tvec.ensure(sizeof(double) * (P->n + 16), st));  // the winner's inlier pass (+ miss, record)
  double* inl_vals = P->tvec.as<double>();
  double* miss = inl_vals + P->n;
  long long* rec = reinterpret_cast<long long*>(inl_vals + P->n + 2);
  const int64_t cap = std::min<int64_t>(nr, kFusedRescoreCap);
  if (skip_refine) {
    CK(launched(launch_argmax(P->counts.as<int>(), r_count, r_begin, 0, sc + 2, P->sms, st, sc)));
    CK(launched(launch_pick_argmax(sc + 2, P->lins.as<int>(), r_begin, P->cand_rows.as<int64_t>(),
                                   P->cand_lins.as<int>(), P->win_c.as<int>(), st)));
    CK(cudaEventRecord(P->ev[2], st));
    CK(cudaEventRecord(P->ev[3], st));
  } else {
    CK(launched(launch_compact(P->counts.as<int>(), P->lins.as<int>(), r_count, r_begin, 0.0,
                               P->cand_rows.as<int64_t>(), P->cand_lins.as<int>(), sc + 3, P->sms,
                               st, sc, q)));
    CK(cudaEventRecord(P->ev[2], st));
    const int nblk = (int)((P->n + screen_threads() - 1) / screen_threads());
    CK(P->partial.ensure(sizeof(double) * nblk * nr, st));
    CK(P->err32.ensure(sizeof(double) * nr, st));
    CK(P->sel.ensure(sizeof(int) * nr, st));
    CK(P->vals.ensure(sizeof(double) * P->n * cap, st));
    CK(P->err64.ensure(sizeof(double) * cap, st));
    const ScoreParams s = score_params(P, rs, code, param);
    CK(launched(launch_screen(s, P->cand_rows.as<int64_t>(), P->cand_lins.as<int>(), nr,
                              P->partial.as<double>(), P->err32.as<double>(), sc + 4, st, sc + 3), 2));
    CK(launched(launch_rescore_compact(P->err32.as<double>(), nr, 0.0, P->sel.as<int>(), sc + 5, st,
                                       sc + 3, sc + 4, screen_tolerance(P, code))));
    CK(launched(launch_exact(s, P->cand_rows.as<int64_t>(), P->cand_lins.as<int>(), P->sel.as<int>(),
                             cap, P->vals.as<double>(), P->err64.as<double>(), st, sc + 5), 2));
    CK(launched(launch_winner(P->err64.as<double>(), P->sel.as<int>(), P->cand_rows.as<int64_t>(),
                              cap, P->win_err.as<double>(), P->win_row.as<int64_t>(),
                              P->win_c.as<int>(), st, nullptr, sc + 5)));
    CK(cudaEventRecord(P->ev[3], st));
  }
  // inlier count of the winner: exact sat_l0 at the bin size (metrics.py:143-150)
  const ScoreParams si = score_params(P, rs, kSatL0, P->bin);
  CK(launched(launch_exact(si, P->cand_rows.as<int64_t>(), P->cand_lins.as<int>(), P->win_c.as<int>(),
                           1, inl_vals, miss, st), 2));
  CK(launched(launch_finalize(sc, P->win_err.as<double>(), P->win_c.as<int>(),
                              P->cand_rows.as<int64_t>(), P->cand_lins.as<int>(),
                              P->counts.as<int>(), r_begin, miss,
                              P->stats.as<unsigned long long>(), rec, st)));
  CK(d2h(P->rec_host, rec, 12 * sizeof(long long), st));
  CK(cudaEventRecord(P->ev[4], st));
  P->pend.active = true;
  P->pend.g = *g;
  P->pend.r_begin = r_begin;
  P->pend.r_count = r_count;
  P->pend.cap = cap;
  P->pend.q = q;
  P->pend.code = code;
  P->pend.param = param;
  P->pend.skip_refine = skip_refine;
  P->pend.stream = stream;
  return DSES_OK;
}

extern "C" int dses_search_wait(dses_plan* P, dses_result* out) {
  TrafficScope ts_(P);
  if (!P || !out) return fail(DSES_E_INVALID, "bad arguments");
  if (!P->pend.active) return fail(DSES_E_INVALID, "no search in flight on this plan");
  std::memset(out, 0, sizeof(*out));
  CK(cudaSetDevice(P->device));
  P->pend.active = false;
  const dses_grid* g = &P->pend.g;
  const int64_t r_begin = P->pend.r_begin, r_count = P->pend.r_count, cap = P->pend.cap;
  const double q = P->pend.q, param = P->pend.param;
  const int code = P->pend.code, skip_refine = P->pend.skip_refine;
  void* stream = P->pend.stream;
  int rc = DSES_OK;
  CK(cudaEventSynchronize(P->ev[4]));
  long long h[12];
  std::memcpy(h, P->rec_host, sizeof h);
  out->mstar = h[0];
  out->candidates_evaluated = h[1];
  out->pairs_evaluated = h[7];
  out->votes = h[8];
  out->rechecks = h[9];
  out->winner_row = -1;
  if (out->candidates_evaluated == 0) return DSES_OK;  // caller raises NoCandidateError
  const int64_t kept = h[2], nsel = h[3];
  if (!skip_refine && nsel > cap) {
    // more near-minimum candidates than the fused tail re-scores: staged path
    double mn32;
    double tol;
    int64_t kept2;
    P->cur_r_begin = r_begin;
    P->cur_r_count = r_count;
    rc = dses_stage_screen(P, q, out->mstar, code, param, &kept2, &mn32, &tol, stream);
    if (rc) return rc;
    double e;
    int64_t row, rescored;
    rc = dses_stage_rescore(P, mn32 + tol, code, param, &e, &row, &rescored, stream);
    if (rc) return rc;
    int64_t lin, cnt;
    rc = dses_stage_row_info(P, row, &lin, &cnt, stream);
    if (rc) return rc;
    double m2;
    rc = dses_pose_error(P, g, row, lin, kSatL0, P->bin, &m2, stream);
    if (rc) return rc;
    h[4] = row; h[5] = lin; h[6] = cnt;
    std::memcpy(&h[10], &e, sizeof e);
    std::memcpy(&h[11], &m2, sizeof m2);
  }
  double best_err, miss_h;
  std::memcpy(&best_err, &h[10], sizeof best_err);
  std::memcpy(&miss_h, &h[11], sizeof miss_h);
  out->winner_row = h[4];
  out->winner_lin = h[5];
  out->winner_count = h[6];
  out->candidates_refined = skip_refine ? 0 : std::max<int64_t>(1, kept);
  out->rescored = skip_refine ? 0 : nsel;
  out->best_error = skip_refine ? miss_h : best_err;
  out->best_inliers = P->n - (int64_t)std::llround(miss_h);
  float ms;
  cudaEventElapsedTime(&ms, P->ev[5], P->ev[6]); out->ms_vote_kernel = ms;
  cudaEventElapsedTime(&ms, P->ev[0], P->ev[1]); out->ms_vote = ms;
  cudaEventElapsedTime(&ms, P->ev[1], P->ev[2]); out->ms_select = ms;
  cudaEventElapsedTime(&ms, P->ev[2], P->ev[3]); out->ms_score = ms;
  cudaEventElapsedTime(&ms, P->ev[0], P->ev[4]); out->ms_total = ms;
  out->launches = P->traffic.launches;
  out->h2d_bytes = P->traffic.h2d;
  out->d2h_bytes = P->traffic.d2h;
  return DSES_OK;
}

extern "C" int dses_search(dses_plan* P, const dses_grid* g, int64_t r_begin, int64_t r_count,
                           double q, int code, double param, int skip_refine, dses_result* out,
                           void* stream) {
  if (!out) return fail(DSES_E_INVALID, "bad arguments");
  std::memset(out, 0, sizeof(*out));
  const int rc = dses_search_async(P, g, r_begin, r_count, q, code, param, skip_refine, stream);
  if (rc) return rc;
  return dses_search_wait(P, out);
}

extern "C" int dses_exhaustive(dses_plan* P, const dses_grid* g, int64_t k_trans,
                               const double t_center[3], int code, double param, dses_result* out,
                               void* stream) {
  TrafficScope ts_(P);
  if (!P || !g || !t_center || !out || k_trans < 0 || code < 0 || code > 4)
    return fail(DSES_E_INVALID, "bad arguments");
  std::memset(out, 0, sizeof(*out));
  CK(cudaSetDevice(P->device));
  cudaStream_t st = (cudaStream_t)stream;
  RotSource rs;
  int rc = set_grid(P, g, &rs, st);
  if (rc) return rc;
  const int64_t nside = 2 * k_trans + 1;
  const int64_t ntrans = nside * nside * nside;
  const int64_t nrot = (2 * g->k + 1) * (2 * g->k + 1) * (2 * g->k + 1);
  if (ntrans >= (1ll << 31)) return fail(DSES_E_INVALID, "translation grid too large");
  const int64_t npose = nrot * ntrans;
  CK(cudaEventRecord(P->ev[0], st));
  // every pose (rotation-major, translation lexicographic: _kernels.py:327-381)
  CK(P->cand_rows.ensure(sizeof(int64_t) * npose, st));
  CK(P->cand_lins.ensure(sizeof(int) * npose, st));
  CK(launched(launch_enumerate_poses(0, npose, ntrans, P->cand_rows.as<int64_t>(),
                                     P->cand_lins.as<int>(), st)));
  ScoreParams s = score_params(P, rs, code, param);
  s.d1 = (int)nside;
  s.d2 = (int)nside;
  s.exh_k = (int)k_trans;
  for (int k = 0; k < 3; ++k) s.tcen[k] = t_center[k];
  // fp32 screen of every pose (chunks), then exact binary64 re-score of the
  // poses within the rigorous screen tolerance of the minimum
  const int64_t chunk = 1 << 20;
  const int nblk = (int)((P->n + screen_threads() - 1) / screen_threads());
  CK(P->partial.ensure(sizeof(double) * nblk * std::min<int64_t>(chunk, npose), st));
  CK(P->err32.ensure(sizeof(double) * npose, st));
  unsigned long long* mb = P->scal.as<unsigned long long>() + 4;
  CK(cudaMemsetAsync(mb, 0x7f, sizeof(unsigned long long), st));
  for (int64_t p0 = 0; p0 < npose; p0 += chunk) {
    const int64_t np = std::min<int64_t>(chunk, npose - p0);
    CK(launched(launch_screen(s, P->cand_rows.as<int64_t>() + p0, P->cand_lins.as<int>() + p0, np,
                              P->partial.as<double>(), P->err32.as<double>() + p0, mb, st),
                (int)((np + 65534) / 65535) + 1));
  }
  double mn;
  CK(d2h(&mn, mb, sizeof mn, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaEventRecord(P->ev[2], st));
  const double thr = mn + screen_tolerance(P, code);
  CK(P->sel.ensure(sizeof(int) * npose, st));
  unsigned long long* ns = P->scal.as<unsigned long long>() + 5;
  CK(cudaMemsetAsync(ns, 0, sizeof(unsigned long long), st));
  CK(launched(launch_rescore_compact(P->err32.as<double>(), npose, thr, P->sel.as<int>(), ns, st)));
  unsigned long long nsel;
  CK(d2h(&nsel, ns, sizeof nsel, st));
  CK(cudaStreamSynchronize(st));
  if (nsel == 0) return fail(DSES_E_CUDA, "internal: exhaustive screen selected no pose");
  CK(P->vals.ensure(sizeof(double) * P->n * nsel, st));
  CK(P->err64.ensure(sizeof(double) * nsel, st));
  CK(P->win_err.ensure(sizeof(double), st));
  CK(P->win_row.ensure(sizeof(int64_t), st));
  CK(P->win_c.ensure(sizeof(int), st));
  CK(launched(launch_exact(s, P->cand_rows.as<int64_t>(), P->cand_lins.as<int>(), P->sel.as<int>(),
                           (int64_t)nsel, P->vals.as<double>(), P->err64.as<double>(), st),
              (int)((nsel + 65534) / 65535) + 1));
  CK(launched(launch_winner(P->err64.as<double>(), P->sel.as<int>(), P->cand_rows.as<int64_t>(),
                            (int64_t)nsel, P->win_err.as<double>(), P->win_row.as<int64_t>(),
                            P->win_c.as<int>(), st, P->cand_lins.as<int>())));
  double e;
  int64_t r;
  int c;
  CK(d2h(&e, P->win_err.p, sizeof e, st));
  CK(d2h(&r, P->win_row.p, sizeof r, st));
  CK(d2h(&c, P->win_c.p, sizeof c, st));
  CK(cudaStreamSynchronize(st));
  int lin = 0;
  CK(d2h(&lin, P->cand_lins.as<int>() + c, sizeof lin, st));
  CK(cudaEventRecord(P->ev[4], st));
  CK(cudaEventSynchronize(P->ev[4]));
  out->candidates_evaluated = npose;
  out->candidates_refined = 0;
  out->winner_row = r;
  out->winner_lin = lin;
  out->best_error = e;
  out->rescored = (int64_t)nsel;
  float ms;
  cudaEventElapsedTime(&ms, P->ev[0], P->ev[2]); out->ms_score = ms;
  cudaEventElapsedTime(&ms, P->ev[0], P->ev[4]); out->ms_total = ms;
  out->launches = P->traffic.launches;
  out->h2d_bytes = P->traffic.h2d;
  out->d2h_bytes = P->traffic.d2h;
  return DSES_OK;
}

// ---- device-resident sharded search ----------------------
// The exchange record x[7] (int64, DEVICE memory of the caller, e.g. a torch
// tensor reduced with NCCL between the calls):
//   x[0] M*          (local, then all_reduce MAX)
//   x[1] error bits  (binary64 bits of the local winner's exact error; the
//                     order of non-negative doubles is their int64 order; MIN)
//   x[2] key         (row << 32 | flat bin of the local winner; MIN after
//                     dses_shard_key masks ranks whose error is not the minimum)
//   x[3] rotations with a vote, x[4] kept candidates, x[5] the winner's
//        sat_l0 miss (binary64 bits, only on the winner's rank),
//   x[6] overflow flag (more near-minimum candidates than the fused tail
//        re-scores: the caller falls back to the staged protocol)  -- SUM
// Local values the later steps compare against stay in the plan's scalars.
namespace {
__global__ void shard_put_vote(const unsigned long long* sc, long long* x) {
  x[0] = (long long)sc[0];
  x[3] = (long long)sc[1];
}
__global__ void shard_get_mstar(unsigned long long* sc, const long long* x) { sc[0] = (unsigned long long)x[0]; }
// sc[8] local error bits, sc[9] local key, sc[10] local miss bits
__global__ void shard_put_select(unsigned long long* sc, const double* win_err, const int* win_c,
                                 const int64_t* cand_rows, const int* cand_lins, const double* miss,
                                 int64_t cap, int skip, long long* x) {
  const int c = *win_c;
  long long eb = LLONG_MAX, key = LLONG_MAX, mb = 0;
  if (c >= 0) {
    const double e = skip ? 0.0 : *win_err;
    eb = __double_as_longlong(e);
    key = (long long)((unsigned long long)cand_rows[c] << 32) | (long long)(unsigned)cand_lins[c];
    mb = __double_as_longlong(*miss);
  }
  sc[8] = (unsigned long long)eb;
  sc[9] = (unsigned long long)key;
  sc[10] = (unsigned long long)mb;
  x[1] = eb;
  x[2] = key;
  x[4] = skip ? 0 : (long long)sc[3];
  x[5] = 0;
  x[6] = (!skip && (long long)sc[5] > cap) ? 1 : 0;
}
__global__ void shard_mask_key(const unsigned long long* sc, long long* x) {
  if ((long long)sc[8] != x[1]) x[2] = LLONG_MAX;
}
__global__ void shard_put_miss(const unsigned long long* sc, long long* x) {
  x[5] = ((long long)sc[9] == x[2]) ? (long long)sc[10] : 0;
}
}  // namespace

extern "C" int dses_shard_vote(dses_plan* P, const dses_grid* g, int64_t r_begin, int64_t r_count,
                               int64_t* xchg, void* stream) {
  TrafficScope ts_(P);
  if (!P || !g || !xchg) return fail(DSES_E_INVALID, "bad arguments");
  if (P->pend.active) return fail(DSES_E_INVALID, "plan has a search in flight");
  CK(cudaSetDevice(P->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t total = (2 * g->k + 1) * (2 * g->k + 1) * (2 * g->k + 1);
  if (r_begin < 0 || r_count < 0 || r_begin + r_count > total)
    return fail(DSES_E_INVALID, "rotation range beyond the grid");
  if (!lattice_fits_int32(P))
    return fail(DSES_E_LIMIT, "translation window of %.3g bins: the search supports lattices "
                "below 2^31 bins", (double)P->dims[0] * P->dims[1] * P->dims[2]);
  int rc = reserve_search(P, std::max<int64_t>(r_count, 1), st);
  if (rc) return rc;
  RotSource rs;
  rc = set_grid(P, g, &rs, st);
  if (rc) return rc;
  P->cur_k = g->k;
  rc = run_vote(P, rs, r_begin, r_count, st);
  if (rc) return rc;
  unsigned long long* sc = P->scal.as<unsigned long long>();
  CK(cudaMemsetAsync(sc, 0, 6 * sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(sc + 2, 0xff, sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(sc + 4, 0x7f, sizeof(unsigned long long), st));
  if (r_count > 0) CK(launched(launch_select_stats(P->counts.as<int>(), r_count, sc, sc + 1, P->sms, st)));
  shard_put_vote<<<1, 1, 0, st>>>(sc, reinterpret_cast<long long*>(xchg));
  CK(launched(cudaGetLastError()));
  return DSES_OK;
}

extern "C" int dses_shard_select(dses_plan* P, double q, int code, double param, int skip_refine,
                                 int64_t* xchg, void* stream) {
  TrafficScope ts_(P);
  if (!P || !xchg || code < 0 || code > 4) return fail(DSES_E_INVALID, "bad arguments");
  CK(cudaSetDevice(P->device));
  cudaStream_t st = (cudaStream_t)stream;
  long long* x = reinterpret_cast<long long*>(xchg);
  const int64_t r_begin = P->cur_r_begin, r_count = P->cur_r_count;
  const int64_t nr = std::max<int64_t>(r_count, 1);
  unsigned long long* sc = P->scal.as<unsigned long long>();
  shard_get_mstar<<<1, 1, 0, st>>>(sc, x);  // the GLOBAL M*
  CK(launched(cudaGetLastError()));
  double* inl_vals = P->tvec.as<double>();
  double* miss = inl_vals + P->n;
  const int64_t cap = std::min<int64_t>(nr, kFusedRescoreCap);
  CK(cudaMemsetAsync(P->win_c.p, 0xff, sizeof(int), st));  // no local winner yet
  if (r_count > 0) {
    const RotSource& rs = P->cur_rot;
    if (skip_refine) {
      CK(cudaMemsetAsync(sc + 2, 0xff, sizeof(unsigned long long), st));
      CK(launched(launch_argmax(P->counts.as<int>(), r_count, r_begin, 0, sc + 2, P->sms, st, sc)));
      CK(launched(launch_pick_argmax(sc + 2, P->lins.as<int>(), r_begin, P->cand_rows.as<int64_t>(),
                                     P->cand_lins.as<int>(), P->win_c.as<int>(), st)));
    } else {
      CK(cudaMemsetAsync(sc + 3, 0, sizeof(unsigned long long), st));
      CK(cudaMemsetAsync(sc + 4, 0x7f, sizeof(unsigned long long), st));
      CK(cudaMemsetAsync(sc + 5, 0, sizeof(unsigned long long), st));
      CK(launched(launch_compact(P->counts.as<int>(), P->lins.as<int>(), r_count, r_begin, 0.0,
                                 P->cand_rows.as<int64_t>(), P->cand_lins.as<int>(), sc + 3, P->sms,
                                 st, sc, q)));
      const ScoreParams s = score_params(P, rs, code, param);
      CK(launched(launch_screen(s, P->cand_rows.as<int64_t>(), P->cand_lins.as<int>(), nr,
                                P->partial.as<double>(), P->err32.as<double>(), sc + 4, st, sc + 3), 2));
      CK(launched(launch_rescore_compact(P->err32.as<double>(), nr, 0.0, P->sel.as<int>(), sc + 5, st,
                                         sc + 3, sc + 4, screen_tolerance(P, code))));
      CK(launched(launch_exact(s, P->cand_rows.as<int64_t>(), P->cand_lins.as<int>(), P->sel.as<int>(),
                               cap, P->vals.as<double>(), P->err64.as<double>(), st, sc + 5), 2));
      CK(launched(launch_winner(P->err64.as<double>(), P->sel.as<int>(), P->cand_rows.as<int64_t>(),
                                cap, P->win_err.as<double>(), P->win_row.as<int64_t>(),
                                P->win_c.as<int>(), st, nullptr, sc + 5)));
    }
    // the local winner's inlier count: exact sat_l0 at the bin size (metrics.py:143-150)
    const ScoreParams si = score_params(P, rs, kSatL0, P->bin);
    CK(launched(launch_exact(si, P->cand_rows.as<int64_t>(), P->cand_lins.as<int>(), P->win_c.as<int>(),
                             1, inl_vals, miss, st), 2));
  }
  shard_put_select<<<1, 1, 0, st>>>(sc, P->win_err.as<double>(), P->win_c.as<int>(),
                                    P->cand_rows.as<int64_t>(), P->cand_lins.as<int>(), miss, cap,
                                    skip_refine, x);
  CK(launched(cudaGetLastError()));
  return DSES_OK;
}

extern "C" int dses_shard_key(dses_plan* P, int64_t* xchg, void* stream) {
  if (!P || !xchg) return fail(DSES_E_INVALID, "bad arguments");
  CK(cudaSetDevice(P->device));
  shard_mask_key<<<1, 1, 0, (cudaStream_t)stream>>>(P->scal.as<unsigned long long>(),
                                                    reinterpret_cast<long long*>(xchg));
  CK(cudaGetLastError());
  return DSES_OK;
}

extern "C" int dses_shard_miss(dses_plan* P, int64_t* xchg, void* stream) {
  if (!P || !xchg) return fail(DSES_E_INVALID, "bad arguments");
  CK(cudaSetDevice(P->device));
  shard_put_miss<<<1, 1, 0, (cudaStream_t)stream>>>(P->scal.as<unsigned long long>(),
                                                    reinterpret_cast<long long*>(xchg));
  CK(cudaGetLastError());
  return DSES_OK;
}

extern "C" int dses_plan_traffic(dses_plan* P, int64_t* h2d_bytes, int64_t* d2h_bytes,
                                 int64_t* launches, int reset) {
  if (!P) return fail(DSES_E_INVALID, "null plan");
  if (h2d_bytes) *h2d_bytes = P->traffic.h2d;
  if (d2h_bytes) *d2h_bytes = P->traffic.d2h;
  if (launches) *launches = P->traffic.launches;
  if (reset) P->traffic = Traffic{};
  return DSES_OK;
}
