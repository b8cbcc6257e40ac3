// Host -> HBM upload of a row-major matrix held in pageable host memory.
//
// The drop-in API takes X as a numpy array (ProblemInstance, model.py:75-116),
// i.e. pageable memory.  A plain cudaMemcpy from pageable memory runs through
// the driver's small bounce buffer on one thread.  Here a pool of host
// threads copies row blocks into pinned staging slots while the copy engine
// streams earlier slots to HBM (cudaMemcpy2DAsync, so the device rows may
// carry a padded pitch).  Every thread owns a pair of slots and walks its own
// blocks (block b belongs to thread b mod T): it waits only for the DMA that
// last read its slot, fills it and queues the transfer itself, so no thread
// ever waits for another one (the first version filled one 16 MB slot with all
// threads between two condition-variable barriers per block: 256 barriers for
// C2's 2 GB, and every block as slow as its slowest thread).

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace l0 {

struct StagingRing {
  static constexpr int kMaxThreads = 32;
  static constexpr int kSlots = 2 * kMaxThreads;   // two per thread
  std::mutex mu;                    // one upload at a time per process
  void* slot[kSlots] = {};
  size_t slot_bytes = 0;
  int nslots = 0;
  cudaEvent_t done[kSlots] = {};
  int device = -1;

  int ensure(size_t bytes, int count, int dev) {
    if (slot_bytes >= bytes && nslots >= count && device == dev) return ST_OK;
    release();
    for (int s = 0; s < count; ++s) {
      if (cudaHostAlloc(&slot[s], bytes, cudaHostAllocPortable) != cudaSuccess)
        return set_error(ST_CUDA, "cudaHostAlloc of the upload staging ring failed");
      if (cudaEventCreateWithFlags(&done[s], cudaEventDisableTiming) != cudaSuccess)
        return set_error(ST_CUDA, "cudaEventCreate failed");
    }
    slot_bytes = bytes;
    nslots = count;
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
    nslots = 0;
  }
};
static StagingRing g_ring;

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
  if (getenv("L0_UPLOAD_THREADS")) threads = atoi(getenv("L0_UPLOAD_THREADS"));
  const int T = std::max(1, std::min<int>(threads > 0 ? threads : 8, StagingRing::kMaxThreads));
  // staging slot size per thread (L0_UPLOAD_MB overrides), two slots per
  // thread; C2's 2 GB (profiles/r2_upload_bw.txt, pinned DMA alone 54.5 GB/s):
  // 4 MB x 8 threads 50.5 GB/s, 2 MB 49.1, 8 MB 50.2, 16 MB 45.7; 12 / 16
  // threads 49.1 / 48.0 (the box has 16 hardware threads)
  const size_t slot_mb = getenv("L0_UPLOAD_MB") ? (size_t)std::max(1, atoi(getenv("L0_UPLOAD_MB"))) : 4;
  const size_t want = std::max<size_t>(slot_mb << 20, (size_t)row_bytes);
  int rc = g_ring.ensure(want, 2 * T, dev);
  if (rc) return rc;
  const int64_t rows_per = std::max<int64_t>(1, (int64_t)(g_ring.slot_bytes / (size_t)row_bytes));
  const int64_t nblocks = (rows + rows_per - 1) / rows_per;
  std::vector<int> err(T, 0);
  std::atomic<int> dma_err{(int)cudaSuccess};
  auto worker = [&](int tid) {
    cudaSetDevice(dev);
    int64_t mine = 0;
    for (int64_t b = tid; b < nblocks; b += T, ++mine) {
      const int slot = 2 * tid + (int)(mine & 1);
      const int64_t r0 = b * rows_per, nr = std::min(rows_per, rows - r0);
      // the slot's previous DMA must have drained before it is refilled
      if (mine >= 2 && cudaEventSynchronize(g_ring.done[slot]) != cudaSuccess) err[tid] = 1;
      char* dst = static_cast<char*>(g_ring.slot[slot]);
      const char* src = static_cast<const char*>(h_src) + r0 * h_pitch;
      if (h_pitch == row_bytes) {
        std::memcpy(dst, src, (size_t)(nr * row_bytes));
      } else {
        for (int64_t r = 0; r < nr; ++r, dst += row_bytes, src += h_pitch)
          std::memcpy(dst, src, (size_t)row_bytes);
      }
      cudaError_t e = cudaMemcpy2DAsync(static_cast<char*>(d_dst) + r0 * d_pitch, (size_t)d_pitch,
                                        g_ring.slot[slot], (size_t)row_bytes, (size_t)row_bytes,
                                        (size_t)nr, cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess) e = cudaEventRecord(g_ring.done[slot], s);
      if (e != cudaSuccess) dma_err.store((int)e);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < T; ++t) pool.emplace_back(worker, t);
  worker(0);
  for (auto& th : pool) th.join();
  if (dma_err.load() != (int)cudaSuccess)
    return set_error(ST_CUDA, std::string("upload: ") + cudaGetErrorString((cudaError_t)dma_err.load()));
  for (int t = 0; t < T; ++t)
    if (err[t]) return set_error(ST_CUDA, "upload: staging event wait failed");
  // the staging slots are reused by the next call: drain before returning
  L0_CUDA_TRY(cudaStreamSynchronize(s));
  return ST_OK;
}
