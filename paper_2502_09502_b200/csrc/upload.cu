// Host -> HBM upload of a row-major matrix held in pageable host memory.
//
// The drop-in API takes X as a numpy array (ProblemInstance, model.py:75-116),
// i.e. pageable memory.  A plain cudaMemcpy from pageable memory runs through
// the driver's small bounce buffer on one thread.  Here a pool of host
// threads copies row blocks into a ring of pinned staging slots while the
// copy engine streams the previous slot to HBM (cudaMemcpy2DAsync, so the
// device rows may carry a padded pitch), i.e. the host memcpy overlaps the
// DMA and is spread over the cores.

#include <algorithm>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace l0 {

struct StagingRing {
  static constexpr int kSlots = 4;
  std::mutex mu;                    // one upload at a time per process
  void* slot[kSlots] = {};
  size_t slot_bytes = 0;
  cudaEvent_t done[kSlots] = {};
  int device = -1;

  int ensure(size_t bytes, int dev) {
    if (slot_bytes >= bytes && device == dev) return ST_OK;
    release();
    for (int s = 0; s < kSlots; ++s) {
      if (cudaHostAlloc(&slot[s], bytes, cudaHostAllocPortable) != cudaSuccess)
        return set_error(ST_CUDA, "cudaHostAlloc of the upload staging ring failed");
      if (cudaEventCreateWithFlags(&done[s], cudaEventDisableTiming) != cudaSuccess)
        return set_error(ST_CUDA, "cudaEventCreate failed");
    }
    slot_bytes = bytes;
    device = dev;
    return ST_OK;
  }
  void release() {
    for (int s = 0; s < kSlots; ++s) {
      if (slot[s]) cudaFreeHost(slot[s]);
      if (done[s]) cudaEventDestroy(done[s]);
      slot[s] = nullptr;
      done[s] = nullptr;
    }
    slot_bytes = 0;
  }
};
static StagingRing g_ring;

// generation barrier for the fill threads
struct Barrier {
  std::mutex m;
  std::condition_variable cv;
  int n, waiting = 0;
  long gen = 0;
  explicit Barrier(int count) : n(count) {}
  void wait() {
    std::unique_lock<std::mutex> lk(m);
    const long g = gen;
    if (++waiting == n) {
      waiting = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

}  // namespace l0

extern "C" int32_t l0_upload_rows(void* d_dst, int64_t d_pitch, const void* h_src, int64_t h_pitch,
                                  int64_t row_bytes, int64_t rows, int32_t threads, void* stream) {
  using namespace l0;
  if (!d_dst || !h_src) return set_error(ST_INVALID, "null argument");
  if (rows < 0 || row_bytes < 0 || d_pitch < row_bytes || h_pitch < row_bytes)
    return set_error(ST_INVALID, "bad upload geometry");
  if (rows == 0 || row_bytes == 0) return ST_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int dev = 0;
  L0_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_ring.mu);
  // staging slot size (L0_UPLOAD_MB overrides; 16 MB measured best for C2's
  // 2 GB: 51 GB/s vs 45.7 at 32 MB and 41 at 128 MB, pinned DMA alone 55.6)
  const size_t slot_mb = getenv("L0_UPLOAD_MB") ? (size_t)std::max(1, atoi(getenv("L0_UPLOAD_MB"))) : 16;
  const size_t want = std::max<size_t>(slot_mb << 20, (size_t)row_bytes);
  int rc = g_ring.ensure(want, dev);
  if (rc) return rc;
  const int64_t rows_per = std::max<int64_t>(1, (int64_t)(g_ring.slot_bytes / (size_t)row_bytes));
  const int64_t nblocks = (rows + rows_per - 1) / rows_per;
  if (getenv("L0_UPLOAD_THREADS")) threads = atoi(getenv("L0_UPLOAD_THREADS"));
  const int T = std::max(1, std::min<int>(threads > 0 ? threads : 8, 32));
  Barrier bar(T);
  std::vector<int> err(T, 0);
  cudaError_t dma_err = cudaSuccess;
  auto worker = [&](int tid) {
    for (int64_t b = 0; b < nblocks; ++b) {
      const int slot = (int)(b % StagingRing::kSlots);
      const int64_t r0 = b * rows_per, nr = std::min(rows_per, rows - r0);
      // the slot's previous DMA must have drained before it is refilled
      if (b >= StagingRing::kSlots && cudaEventSynchronize(g_ring.done[slot]) != cudaSuccess)
        err[tid] = 1;
      // rows of this block split over the threads (contiguous spans)
      const int64_t a0 = r0 + nr * tid / T, a1 = r0 + nr * (tid + 1) / T;
      char* dst = static_cast<char*>(g_ring.slot[slot]) + (a0 - r0) * row_bytes;
      const char* src = static_cast<const char*>(h_src) + a0 * h_pitch;
      if (h_pitch == row_bytes) {
        std::memcpy(dst, src, (size_t)((a1 - a0) * row_bytes));
      } else {
        for (int64_t r = a0; r < a1; ++r, dst += row_bytes, src += h_pitch)
          std::memcpy(dst, src, (size_t)row_bytes);
      }
      bar.wait();
      if (tid == 0) {
        cudaError_t e = cudaMemcpy2DAsync(static_cast<char*>(d_dst) + r0 * d_pitch, (size_t)d_pitch,
                                          g_ring.slot[slot], (size_t)row_bytes, (size_t)row_bytes,
                                          (size_t)nr, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaEventRecord(g_ring.done[slot], s);
        if (e != cudaSuccess) dma_err = e;
      }
      bar.wait();   // the event is recorded before anyone waits on it
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < T; ++t) pool.emplace_back(worker, t);
  worker(0);
  for (auto& th : pool) th.join();
  if (dma_err != cudaSuccess) return set_error(ST_CUDA, std::string("upload: ") + cudaGetErrorString(dma_err));
  for (int t = 0; t < T; ++t)
    if (err[t]) return set_error(ST_CUDA, "upload: staging event wait failed");
  // the staging slots are reused by the next call: drain before returning
  L0_CUDA_TRY(cudaStreamSynchronize(s));
  return ST_OK;
}
