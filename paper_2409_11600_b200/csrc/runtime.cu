// libnskb runtime: errors, device init, the size-class caching allocator,
// pinned staging, streams/events, CUDA graphs and TMA descriptor encoding.
//
// The device allocator is the backing store for the Python-level Pool
// (reference: pkg/src/nsk/tensor.py:54-113). The Pool keeps the reference's
// exact-numel LIFO semantics and statistics; fresh acquisitions land here,
// where requests are rounded to size classes and recycled stream-ordered, so
// a cudaMalloc happens only when no cached block of the class is free.
#include <mutex>
#include <unordered_map>
#include <map>
#include <vector>
#include <cstring>
#include <cstdio>

#include "common.cuh"
#include "../../include/nskb.h"

namespace nsk {

static thread_local std::string g_last_error;
static int g_sm_count = 0;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return set_error(NSK_ERR_OOM, std::string("out of memory in ") + where);
  }
  return set_error(NSK_ERR_CUDA, std::string(cudaGetErrorString(e)) + " in " + where);
}

int sm_count() {
  if (g_sm_count == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    g_sm_count = n;
  }
  return g_sm_count;
}

int grid_cap_per_sm() {
  static int cap = -1;
  if (cap < 0) {
    const char* e = getenv("NSK_GRID_CAP");
    cap = e ? atoi(e) : 16;
    if (cap < 1) cap = 16;
  }
  return cap;
}

bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("NSK_PDL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// ---- TMA descriptor encoding --------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn g_encode = nullptr;

int encode_tmap(CUtensorMap* map, CUtensorMapDataType dt, int rank, const void* gaddr, const uint64_t* dims,
                const uint64_t* strides_bytes, const uint32_t* box, const uint32_t* elem_strides,
                CUtensorMapSwizzle swz) {
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || fn == nullptr) return set_error(NSK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    g_encode = (EncodeTiledFn)fn;
  }
  cuuint64_t d[5], s[5];
  cuuint32_t b[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    es[i] = elem_strides ? elem_strides[i] : 1;
    if (i < rank - 1) s[i] = strides_bytes[i];
  }
  CUresult r = g_encode(map, dt, (cuuint32_t)rank, const_cast<void*>(gaddr), d, s, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[256];
    snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d): rank %d dims %llu,%llu,%llu,%llu box %u,%u,%u,%u",
             (int)r, rank, (unsigned long long)d[0], (unsigned long long)(rank > 1 ? d[1] : 0),
             (unsigned long long)(rank > 2 ? d[2] : 0), (unsigned long long)(rank > 3 ? d[3] : 0), b[0],
             rank > 1 ? b[1] : 0, rank > 2 ? b[2] : 0, rank > 3 ? b[3] : 0);
    return set_error(NSK_ERR_SHAPE, buf);
  }
  return NSK_OK;
}

typedef CUresult (*EncodeIm2colFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeIm2colFn g_encode_i2c = nullptr;

int encode_tmap_im2col(CUtensorMap* map, const void* gaddr, int N, int H, int W, int C, const int* lower_wh,
                       const int* upper_wh, int pixels, int stride) {
  if (!g_encode_i2c) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || fn == nullptr) return set_error(NSK_ERR_CUDA, "cuTensorMapEncodeIm2col unavailable");
    g_encode_i2c = (EncodeIm2colFn)fn;
  }
  cuuint64_t d[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t s[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
  cuuint32_t es[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
  CUresult r = g_encode_i2c(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(gaddr), d, s, lower_wh,
                            upper_wh, 64, (cuuint32_t)pixels, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[256];
    snprintf(buf, sizeof buf,
             "cuTensorMapEncodeIm2col failed (%d): NHWC %d,%d,%d,%d corners (%d,%d)..(%d,%d) pixels %d stride %d",
             (int)r, N, H, W, C, lower_wh[0], lower_wh[1], upper_wh[0], upper_wh[1], pixels, stride);
    return set_error(NSK_ERR_SHAPE, buf);
  }
  // Drivers up to 13.1 mis-handle a descriptor flag for im2col maps over tensors below 128 KiB (the same
  // adjustment CUTLASS applies in copy_traits_sm90_im2col.hpp); clear it for small tensors.
  int drv = 0;
  cudaDriverGetVersion(&drv);
  if (drv <= 13010 && (uint64_t)N * H * W * C * 2 < 131072) reinterpret_cast<uint64_t*>(map)[1] &= ~(1ull << 21);
  return NSK_OK;
}

// ---- caching allocator ---------------------------------------------------------
struct Block {
  size_t size;          // class size (bytes actually reserved)
  cudaStream_t stream;  // stream of last use
  cudaEvent_t ready;    // recorded at free; reuse from another stream waits on it
  bool event_live;
};

class Arena {
 public:
  int alloc(size_t bytes, cudaStream_t stream, void** out) {
    size_t cls = size_class(bytes);
    std::lock_guard<std::mutex> g(mu_);
    auto range = free_.equal_range(cls);
    // prefer a block last used on the same stream (no sync needed)
    for (auto it = range.first; it != range.second; ++it) {
      Block& b = blocks_[it->second];
      if (b.stream == stream || !b.event_live || cudaEventQuery(b.ready) == cudaSuccess) {
        void* p = it->second;
        free_.erase(it);
        b.stream = stream;
        in_use_ += cls;
        ++hits_;
        *out = p;
        return NSK_OK;
      }
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, cls);
    if (e != cudaSuccess) {
      cudaGetLastError();
      release_cached_locked();
      e = cudaMalloc(&p, cls);
      if (e != cudaSuccess) {
        cudaGetLastError();
        char buf[128];
        snprintf(buf, sizeof buf, "out of memory: requested %zu bytes", bytes);
        return set_error(NSK_ERR_OOM, buf);
      }
    }
    Block b{cls, stream, nullptr, false};
    blocks_[p] = b;
    reserved_ += cls;
    in_use_ += cls;
    ++mallocs_;
    *out = p;
    return NSK_OK;
  }

  int free(void* p, cudaStream_t stream) {
    if (!p) return NSK_OK;
    std::lock_guard<std::mutex> g(mu_);
    auto it = blocks_.find(p);
    if (it == blocks_.end()) return set_error(NSK_ERR_RANGE, "free of a pointer the arena does not own");
    Block& b = it->second;
    if (!b.ready) {
      if (cudaEventCreateWithFlags(&b.ready, cudaEventDisableTiming) != cudaSuccess) b.ready = nullptr;
    }
    b.stream = stream;
    b.event_live = false;
    if (b.ready) {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      cudaStreamIsCapturing(stream, &cs);
      if (cs == cudaStreamCaptureStatusNone && cudaEventRecord(b.ready, stream) == cudaSuccess) b.event_live = true;
    }
    in_use_ -= b.size;
    free_.emplace(b.size, p);
    return NSK_OK;
  }

  void stats(uint64_t* out) {
    std::lock_guard<std::mutex> g(mu_);
    out[0] = reserved_;
    out[1] = in_use_;
    out[2] = mallocs_;
    out[3] = hits_;
  }

  int trim() {
    std::lock_guard<std::mutex> g(mu_);
    return release_cached_locked();
  }

 private:
  static size_t size_class(size_t bytes) {
    if (bytes == 0) bytes = 1;
    if (bytes <= (1u << 20)) return (bytes + 511) & ~(size_t)511;
    const size_t two_mb = (size_t)2 << 20;
    return (bytes + two_mb - 1) & ~(two_mb - 1);
  }
  int release_cached_locked() {
    cudaDeviceSynchronize();
    for (auto& kv : free_) {
      auto it = blocks_.find(kv.second);
      if (it != blocks_.end()) {
        if (it->second.ready) cudaEventDestroy(it->second.ready);
        reserved_ -= it->second.size;
        blocks_.erase(it);
      }
      cudaFree(kv.second);
    }
    free_.clear();
    return NSK_OK;
  }

  std::mutex mu_;
  std::unordered_map<void*, Block> blocks_;
  std::multimap<size_t, void*> free_;
  uint64_t reserved_ = 0, in_use_ = 0, mallocs_ = 0, hits_ = 0;
};

static Arena& arena() {
  static Arena* a = new Arena();  // leaked on purpose: outlives static destructors
  return *a;
}

}  // namespace nsk

using namespace nsk;

namespace {
// holds the stream for ns nanoseconds of device time (measurement: lets the host enqueue a whole eager step so its
// kernels then run back to back, without host launch gaps inside event brackets)
__global__ void spin_kernel(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}
}  // namespace

extern "C" {

int nsk_spin(uint64_t ns, void* stream) {
  spin_kernel<<<1, 32, 0, (cudaStream_t)stream>>>((unsigned long long)ns);
  NSK_CUDA(cudaGetLastError());
  return NSK_OK;
}

const char* nsk_last_error(void) { return g_last_error.c_str(); }

int nsk_abi_version(void) { return NSK_ABI_VERSION; }

int nsk_init(int device) {
  NSK_CUDA(cudaSetDevice(device));
  NSK_CUDA(cudaFree(0));
  g_sm_count = 0;
  sm_count();
  return NSK_OK;
}

int nsk_device_info(int* sm_count_out, int* cc_major, int* cc_minor, uint64_t* total_mem) {
  int dev = 0;
  NSK_CUDA(cudaGetDevice(&dev));
  cudaDeviceProp p;
  NSK_CUDA(cudaGetDeviceProperties(&p, dev));
  *sm_count_out = p.multiProcessorCount;
  *cc_major = p.major;
  *cc_minor = p.minor;
  *total_mem = p.totalGlobalMem;
  return NSK_OK;
}

int nsk_arena_alloc(uint64_t bytes, void* stream, void** out) {
  return arena().alloc((size_t)bytes, (cudaStream_t)stream, out);
}
int nsk_arena_free(void* ptr, void* stream) { return arena().free(ptr, (cudaStream_t)stream); }
int nsk_arena_stats(uint64_t* out4) {
  arena().stats(out4);
  return NSK_OK;
}
int nsk_arena_trim(void) { return arena().trim(); }

int nsk_pinned_alloc(uint64_t bytes, void** out) {
  NSK_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable));
  return NSK_OK;
}
int nsk_pinned_free(void* p) {
  NSK_CUDA(cudaFreeHost(p));
  return NSK_OK;
}

int nsk_memcpy_h2d(void* dst, const void* src, uint64_t bytes, void* stream) {
  NSK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream));
  return NSK_OK;
}
int nsk_memcpy_d2h(void* dst, const void* src, uint64_t bytes, void* stream) {
  NSK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  return NSK_OK;
}
int nsk_memcpy_d2d(void* dst, const void* src, uint64_t bytes, void* stream) {
  NSK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return NSK_OK;
}

int nsk_memcpy2d_d2d(void* dst, uint64_t dpitch, const void* src, uint64_t spitch, uint64_t width, uint64_t rows,
                     void* stream) {
  NSK_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return NSK_OK;
}

int nsk_stream_create(void** out) {
  cudaStream_t s;
  NSK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *out = (void*)s;
  return NSK_OK;
}
int nsk_stream_destroy(void* s) {
  NSK_CUDA(cudaStreamDestroy((cudaStream_t)s));
  return NSK_OK;
}
int nsk_stream_sync(void* s) {
  NSK_CUDA(cudaStreamSynchronize((cudaStream_t)s));
  return NSK_OK;
}
int nsk_device_sync(void) {
  NSK_CUDA(cudaDeviceSynchronize());
  return NSK_OK;
}
int nsk_event_create(int timing, void** out) {
  cudaEvent_t e;
  NSK_CUDA(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
  *out = (void*)e;
  return NSK_OK;
}
int nsk_event_destroy(void* e) {
  NSK_CUDA(cudaEventDestroy((cudaEvent_t)e));
  return NSK_OK;
}
int nsk_event_record(void* e, void* stream) {
  NSK_CUDA(cudaEventRecord((cudaEvent_t)e, (cudaStream_t)stream));
  return NSK_OK;
}
// a record that stays a real event-record node when the stream is being captured (cudaEventRecordExternal):
// timing a kernel inside a replayed step graph
int nsk_event_record_external(void* e, void* stream) {
  NSK_CUDA(cudaEventRecordWithFlags((cudaEvent_t)e, (cudaStream_t)stream, cudaEventRecordExternal));
  return NSK_OK;
}
int nsk_event_wait(void* stream, void* e) {
  NSK_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)e, 0));
  return NSK_OK;
}
int nsk_event_sync(void* e) {
  NSK_CUDA(cudaEventSynchronize((cudaEvent_t)e));
  return NSK_OK;
}
int nsk_event_elapsed_ms(void* start, void* stop, float* ms) {
  NSK_CUDA(cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)stop));
  return NSK_OK;
}

int nsk_graph_begin(void* stream) {
  NSK_CUDA(cudaStreamBeginCapture((cudaStream_t)stream, cudaStreamCaptureModeThreadLocal));
  return NSK_OK;
}
int nsk_graph_end(void* stream, void** exec_out, uint64_t* num_nodes) {
  cudaGraph_t g;
  NSK_CUDA(cudaStreamEndCapture((cudaStream_t)stream, &g));
  size_t n = 0;
  cudaGraphGetNodes(g, nullptr, &n);
  if (num_nodes) *num_nodes = n;
  cudaGraphExec_t ex;
  cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_status(e, "cudaGraphInstantiate");
  *exec_out = (void*)ex;
  return NSK_OK;
}
int nsk_graph_launch(void* exec, void* stream) {
  NSK_CUDA(cudaGraphLaunch((cudaGraphExec_t)exec, (cudaStream_t)stream));
  return NSK_OK;
}
int nsk_graph_destroy(void* exec) {
  NSK_CUDA(cudaGraphExecDestroy((cudaGraphExec_t)exec));
  return NSK_OK;
}
int nsk_stream_is_capturing(void* stream, int* out) {
  cudaStreamCaptureStatus cs;
  NSK_CUDA(cudaStreamIsCapturing((cudaStream_t)stream, &cs));
  *out = cs == cudaStreamCaptureStatusActive ? 1 : 0;
  return NSK_OK;
}

}  // extern "C"
