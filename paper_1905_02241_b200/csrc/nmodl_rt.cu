// libnmodl_b200_rt.so -- the C-ABI runtime under every generated mechanism.
//
// Plain pointers and sizes only (declared in include/nmodl_b200.h).  Python
// binds it with ctypes (paper_1905_02241_b200/runtime.py); no PyTorch types
// cross this boundary.  It owns what the reference leaves to "the simulator"
// (modlc/codegen.py:59 "independent iterations"): device
// memory for the SoA instance store, streams, CUDA-graph capture of the
// per-timestep launch loop, the device status block, finiteness scans,
// deterministic checksums for cross-GPU validation, and the node_index
// scatter layout (stable counting sort by node).
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "nmodl_b200/status.h"

#define NMODL_API extern "C" __attribute__((visibility("default")))

static thread_local char g_err[512];

static int fail(cudaError_t e, const char* what) {
  snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
  return (int)e;
}
#define CK(call)                                   \
  do {                                             \
    cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return fail(e_, #call); \
  } while (0)

NMODL_API const char* nmodl_last_error(void) { return g_err; }
NMODL_API int nmodl_abi_version(void) { return 1; }

// ---------------------------------------------------------------------------
// device / memory / streams

NMODL_API int nmodl_device_count(int* out) {
  CK(cudaGetDeviceCount(out));
  return 0;
}
NMODL_API int nmodl_get_device(int* dev) {
  CK(cudaGetDevice(dev));
  return 0;
}
NMODL_API int nmodl_set_device(int dev) {
  CK(cudaSetDevice(dev));
  return 0;
}
NMODL_API int nmodl_device_info(int dev, int* sm_count, long long* l2_bytes, long long* mem_bytes,
                                int* cc_major, int* cc_minor, char* name, int name_len) {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, dev));
  *sm_count = p.multiProcessorCount;
  *l2_bytes = p.l2CacheSize;
  *mem_bytes = (long long)p.totalGlobalMem;
  *cc_major = p.major;
  *cc_minor = p.minor;
  if (name && name_len > 0) {
    strncpy(name, p.name, name_len - 1);
    name[name_len - 1] = 0;
  }
  return 0;
}
NMODL_API int nmodl_malloc(void** out, size_t bytes) {
  CK(cudaMalloc(out, bytes ? bytes : 256));
  return 0;
}
NMODL_API int nmodl_free(void* p) {
  CK(cudaFree(p));
  return 0;
}
NMODL_API int nmodl_host_alloc(void** out, size_t bytes) {
  CK(cudaHostAlloc(out, bytes ? bytes : 64, cudaHostAllocPortable));
  return 0;
}
NMODL_API int nmodl_host_free(void* p) {
  CK(cudaFreeHost(p));
  return 0;
}
NMODL_API int nmodl_host_register(void* p, size_t bytes) {
  CK(cudaHostRegister(p, bytes, cudaHostRegisterPortable));
  return 0;
}
NMODL_API int nmodl_host_unregister(void* p) {
  CK(cudaHostUnregister(p));
  return 0;
}
NMODL_API int nmodl_memcpy_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
  return 0;
}
NMODL_API int nmodl_memcpy_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
  return 0;
}
NMODL_API int nmodl_memcpy_d2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
  return 0;
}
NMODL_API int nmodl_memset(void* dst, int value, size_t bytes, cudaStream_t s) {
  CK(cudaMemsetAsync(dst, value, bytes, s));
  return 0;
}
NMODL_API int nmodl_stream_create(cudaStream_t* out) {
  CK(cudaStreamCreateWithFlags(out, cudaStreamNonBlocking));
  return 0;
}
NMODL_API int nmodl_stream_destroy(cudaStream_t s) {
  CK(cudaStreamDestroy(s));
  return 0;
}
NMODL_API int nmodl_stream_sync(cudaStream_t s) {
  CK(cudaStreamSynchronize(s));
  return 0;
}
NMODL_API int nmodl_device_sync(void) {
  CK(cudaDeviceSynchronize());
  return 0;
}
NMODL_API int nmodl_event_create(cudaEvent_t* out) {
  CK(cudaEventCreate(out));
  return 0;
}
NMODL_API int nmodl_event_destroy(cudaEvent_t e) {
  CK(cudaEventDestroy(e));
  return 0;
}
NMODL_API int nmodl_event_record(cudaEvent_t e, cudaStream_t s) {
  CK(cudaEventRecord(e, s));
  return 0;
}
// Inside a stream capture this becomes an event-record node that keeps its
// timestamp (cudaEventRecordExternal), so kernel boundaries inside a replayed
// graph can be timed; outside a capture it is an ordinary record.
NMODL_API int nmodl_event_record_external(cudaEvent_t e, cudaStream_t s) {
  CK(cudaEventRecordWithFlags(e, s, cudaEventRecordExternal));
  return 0;
}
NMODL_API int nmodl_stream_wait_event(cudaStream_t s, cudaEvent_t e) {
  CK(cudaStreamWaitEvent(s, e, 0));
  return 0;
}
NMODL_API int nmodl_event_sync(cudaEvent_t e) {
  CK(cudaEventSynchronize(e));
  return 0;
}
NMODL_API int nmodl_event_elapsed_ms(cudaEvent_t a, cudaEvent_t b, float* ms) {
  CK(cudaEventElapsedTime(ms, a, b));
  return 0;
}

// ---------------------------------------------------------------------------
// CUDA graphs: the per-timestep launch loop (one kernel per step, v exogenous
// between steps) is captured once and replayed, removing host launch cost.

NMODL_API int nmodl_capture_begin(cudaStream_t s) {
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  return 0;
}
NMODL_API int nmodl_capture_end(cudaStream_t s, cudaGraphExec_t* out) {
  cudaGraph_t g;
  CK(cudaStreamEndCapture(s, &g));
  cudaError_t e = cudaGraphInstantiate(out, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return fail(e, "cudaGraphInstantiate");
  return 0;
}
// upload an instantiated graph's work descriptors to the device ahead of its
// first launch (otherwise the first replay pays for it: ~10 us per step of a
// 200-step, 800-node column graph)
NMODL_API int nmodl_graph_upload(cudaGraphExec_t g, cudaStream_t s) {
  CK(cudaGraphUpload(g, s));
  return 0;
}
NMODL_API int nmodl_graph_launch(cudaGraphExec_t g, cudaStream_t s) {
  CK(cudaGraphLaunch(g, s));
  return 0;
}
NMODL_API int nmodl_graph_destroy(cudaGraphExec_t g) {
  CK(cudaGraphExecDestroy(g));
  return 0;
}

// ---------------------------------------------------------------------------
// status block

NMODL_API int nmodl_status_reset(nmodl_status* st, cudaStream_t s) {
  nmodl_status h;
  h.err_key = NMODL_NO_ERROR;
  h.payload_key = NMODL_NO_ERROR;
  h.payload = 0.0;
  h.lock = 0;
  h.reserved = 0;
  CK(cudaMemcpyAsync(st, &h, sizeof(h), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  return 0;
}
NMODL_API int nmodl_status_size(void) { return (int)sizeof(nmodl_status); }

// ---------------------------------------------------------------------------
// finiteness scan: first non-finite index of an array (atomicMin), used once
// at upload so that pre-existing NaN/Inf in never-written slots are reported
// like the reference's whole-store scan (modlc/interp.py:538-545).

__global__ void k_first_nonfinite(const double* __restrict__ p, long long n,
                                  unsigned long long* out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  for (; i < n; i += stride)
    if (!isfinite(p[i])) atomicMin(out, (unsigned long long)i);
}
NMODL_API int nmodl_first_nonfinite(const double* p, long long n, unsigned long long* out_dev,
                                    cudaStream_t s) {
  if (n <= 0) return 0;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_first_nonfinite<<<blocks, 256, 0, s>>>(p, n, out_dev);
  CK(cudaGetLastError());
  return 0;
}

// ---------------------------------------------------------------------------
// deterministic checksums (fixed reduction tree, independent of launch
// timing) for cross-rank validation: out[0] = sum(x), out[1] = sum(|x|).

__global__ void k_checksum_partial(const double* __restrict__ p, long long n, double* part) {
  __shared__ double s0[256], s1[256];
  double a = 0.0, b = 0.0;
  for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
    double x = p[i];
    a += x;
    b += fabs(x);
  }
  s0[threadIdx.x] = a;
  s1[threadIdx.x] = b;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      s0[threadIdx.x] += s0[threadIdx.x + w];
      s1[threadIdx.x] += s1[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s0[0];
    part[2 * blockIdx.x + 1] = s1[0];
  }
}
__global__ void k_checksum_final(const double* part, int nb, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int i = 0; i < nb; ++i) {
      a += part[2 * i];
      b += part[2 * i + 1];
    }
    out[0] = a;
    out[1] = b;
  }
}
NMODL_API int nmodl_checksum(const double* p, long long n, double* scratch_dev /* >= 2*1024 */,
                             double* out_dev /* 2 */, cudaStream_t s) {
  const int nb = 1024;
  k_checksum_partial<<<nb, 256, 0, s>>>(p, n, scratch_dev);
  k_checksum_final<<<1, 32, 0, s>>>(scratch_dev, nb, out_dev);
  CK(cudaGetLastError());
  return 0;
}

// ---------------------------------------------------------------------------
// L2 flush between timed iterations (write a buffer larger than L2).

__global__ void k_fill(double* p, long long n, double v) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}
NMODL_API int nmodl_l2_flush(double* buf, long long n_doubles, cudaStream_t s) {
  k_fill<<<148 * 8, 256, 0, s>>>(buf, n_doubles, 0.0);
  CK(cudaGetLastError());
  return 0;
}

// After a write flush: read a second buffer larger than L2, so the flush's
// own dirty lines are written back now rather than while the next timed
// kernel runs (L2 ends full of clean lines that hold none of its data).
__global__ void k_read(const double* __restrict__ p, long long n) {
  double acc = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    acc += __ldcg(p + i);
  if (acc == 1.2345e300) asm volatile("trap;");  // never true (buffer is zero): keeps the loads
}
NMODL_API int nmodl_l2_clean(const double* buf, long long n_doubles, cudaStream_t s) {
  k_read<<<148 * 8, 256, 0, s>>>(buf, n_doubles);
  CK(cudaGetLastError());
  return 0;
}

// Device-side head start for host-issued timed sequences: one thread spins
// on %globaltimer for `ns`, so the host can enqueue the events and launches
// that follow before the GPU reaches them (no host gaps inside the timing).
__global__ void k_spin(long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while ((long long)(t - t0) < ns);
}
NMODL_API int nmodl_spin(long long ns, cudaStream_t s) {
  k_spin<<<1, 1, 0, s>>>(ns);
  CK(cudaGetLastError());
  return 0;
}

// ---------------------------------------------------------------------------
// node_index scatter layout (builder-defined extension; the reference has no
// node arrays).  Stable counting sort of instances by node:
//   counts[node]  = #instances on node
//   offsets[0..N] = exclusive scan of counts
//   perm[k]       = k-th instance in (node, instance) order   (stable)
//   rank[i]       = position of instance i in that order (inverse of perm)
// Stability is obtained without atomics-order dependence: every instance's
// rank within its node is the number of equal-node instances before it,
// computed per node segment after a histogram -- deterministic by
// construction and bit-identical to np.argsort(node_index, kind="stable").

__global__ void k_hist(const int* __restrict__ node_index, long long n, int n_nodes,
                       unsigned int* counts, int* bad) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int nd = node_index[i];
    if (nd < 0 || nd >= n_nodes) {
      atomicMin(bad, (int)(i < 0x7fffffff ? i : 0x7fffffff));
      continue;
    }
    atomicAdd(&counts[nd], 1u);
  }
}

// counts (u32) -> int64 with a trailing zero so an exclusive scan over n+1
// entries yields offsets[n_nodes] = total
__global__ void k_widen(const unsigned int* counts, int n_nodes, long long* out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i <= n_nodes;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = i < n_nodes ? (long long)counts[i] : 0;
}

// Stable placement: CUB's LSD radix sort of (node, instance) pairs is stable,
// so equal nodes keep ascending instance order -- bit-identical to
// np.argsort(node_index, kind="stable").  Setup-time only.
__global__ void k_iota_rank(long long* iota, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    iota[i] = i;
}
__global__ void k_invert(const long long* __restrict__ perm, long long* __restrict__ rank,
                         long long n) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x)
    rank[perm[k]] = k;
}

// Keep the stream-ordered allocator's pool across synchronisations: with the
// default release threshold (0) every sync hands the memory back to the
// driver and the next cudaMallocAsync of CUB's scratch pays for it again.
static void keep_async_pool() {
  static bool done = false;
  if (done) return;
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    unsigned long long threshold = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
  }
  done = true;
}

NMODL_API int nmodl_scatter_layout(const int* node_index_dev, long long n, int n_nodes,
                                   unsigned int* counts_dev /* n_nodes */,
                                   long long* offsets_dev /* n_nodes + 1 */,
                                   long long* scratch_dev /* n */, long long* perm_dev /* n */,
                                   long long* rank_dev /* n */, int* bad_dev /* 1 */,
                                   cudaStream_t s) {
  keep_async_pool();
  CK(cudaMemsetAsync(counts_dev, 0, sizeof(unsigned int) * (size_t)n_nodes, s));
  int big = 0x7fffffff;
  CK(cudaMemcpyAsync(bad_dev, &big, sizeof(int), cudaMemcpyHostToDevice, s));
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  k_hist<<<blocks, 256, 0, s>>>(node_index_dev, n, n_nodes, counts_dev, bad_dev);
  // offsets[0..n_nodes] = exclusive scan of counts (int64), via CUB
  k_widen<<<blocks, 256, 0, s>>>(counts_dev, n_nodes, offsets_dev);
  {
    size_t scan_bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, offsets_dev, offsets_dev, (int64_t)n_nodes + 1, s));
    void* scan_tmp = nullptr;
    CK(cudaMallocAsync(&scan_tmp, scan_bytes ? scan_bytes : 16, s));
    CK(cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, offsets_dev, offsets_dev, (int64_t)n_nodes + 1, s));
    CK(cudaFreeAsync(scan_tmp, s));
  }
  k_iota_rank<<<blocks, 256, 0, s>>>(scratch_dev, n);
  int* keys_out = nullptr;
  CK(cudaMallocAsync((void**)&keys_out, sizeof(int) * (size_t)(n > 0 ? n : 1), s));
  int end_bit = 1;
  while (end_bit < 31 && (1 << end_bit) < n_nodes) ++end_bit;
  size_t temp_bytes = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, node_index_dev, keys_out, scratch_dev,
                                     perm_dev, (int64_t)n, 0, end_bit, s));
  void* temp = nullptr;
  CK(cudaMallocAsync(&temp, temp_bytes ? temp_bytes : 16, s));
  CK(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, node_index_dev, keys_out, scratch_dev,
                                     perm_dev, (int64_t)n, 0, end_bit, s));
  k_invert<<<blocks, 256, 0, s>>>(perm_dev, rank_dev, n);
  CK(cudaFreeAsync(temp, s));
  CK(cudaFreeAsync(keys_out, s));
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  return 0;
}

// occupied segments and CTA tiles of a node layout, on the device
// (runner.bind_nodes; the host restatement is runner.tile_nodes_for):
//   seg_node = nodes k with offsets[k+1] > offsets[k], ascending
//   seg_off  = offsets[seg_node] ++ [n]
//   tiles    = unique([0] ++ lower_bound(seg_off[:-1], m*T for m*T < max(n,1)) ++ [n_segs])
__global__ void k_seg_flags(const long long* __restrict__ offsets, int n_nodes, unsigned char* __restrict__ flag) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n_nodes;
       k += (long long)gridDim.x * blockDim.x)
    flag[k] = offsets[k + 1] > offsets[k] ? 1 : 0;
}
__global__ void k_seg_offsets(const long long* __restrict__ offsets, const int* __restrict__ seg_node,
                              const long long* __restrict__ n_segs_dev, long long n, long long* __restrict__ seg_off) {
  const long long m = *n_segs_dev;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j <= m;
       j += (long long)gridDim.x * blockDim.x)
    seg_off[j] = j < m ? offsets[seg_node[j]] : n;
}
__global__ void k_tile_marks(const long long* __restrict__ seg_off, const long long* __restrict__ n_segs_dev,
                             long long n_marks, long long tile, long long* __restrict__ cand,
                             unsigned char* __restrict__ flag) {
  const long long m = *n_segs_dev;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t <= n_marks;
       t += (long long)gridDim.x * blockDim.x) {
    long long c;
    if (t == n_marks) {
      c = m;
    } else {  // first segment whose offset is >= t * tile
      const long long key = t * tile;
      long long lo = 0, hi = m;
      while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (seg_off[mid] < key) lo = mid + 1; else hi = mid;
      }
      c = lo;
    }
    cand[t] = c;
  }
}
__global__ void k_tile_flags(const long long* __restrict__ cand, long long n_cand, unsigned char* __restrict__ flag) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n_cand;
       t += (long long)gridDim.x * blockDim.x)
    flag[t] = (t == 0 || cand[t] != cand[t - 1]) ? 1 : 0;
}

static int grid_for(long long n) {
  long long b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return b < 1 ? 1 : (int)b;
}

NMODL_API int nmodl_node_segments(const long long* offsets_dev /* n_nodes + 1 */, int n_nodes, long long n,
                                  long long tile, int* seg_node_dev /* n_nodes */,
                                  long long* seg_off_dev /* n_nodes + 1 */,
                                  long long* tiles_dev /* n_marks + 2, n_marks = ceil(max(n,1)/tile) */,
                                  long long* counts_dev /* 2: n_segs, n_tiles + 1 */, cudaStream_t s) {
  keep_async_pool();
  if (tile < 1) return (int)cudaErrorInvalidValue;
  const long long n_marks = ((n > 0 ? n : 1) + tile - 1) / tile;
  // marks start at 0, so cand[0] = 0 and the leading [0] of the restatement is implicit
  const long long n_cand = n_marks + 1;
  unsigned char* flag = nullptr;
  long long* cand = nullptr;
  const long long flag_len = (n_nodes > n_cand ? (long long)n_nodes : n_cand) + 1;
  CK(cudaMallocAsync((void**)&flag, (size_t)flag_len, s));
  CK(cudaMallocAsync((void**)&cand, sizeof(long long) * (size_t)n_cand, s));
  k_seg_flags<<<grid_for(n_nodes), 256, 0, s>>>(offsets_dev, n_nodes, flag);
  size_t bytes = 0, b2 = 0;
  CK(cub::DeviceSelect::Flagged(nullptr, bytes, cub::CountingInputIterator<int>(0), flag, seg_node_dev,
                                counts_dev, n_nodes, s));
  CK(cub::DeviceSelect::Flagged(nullptr, b2, cand, flag, tiles_dev, counts_dev + 1, n_cand, s));
  if (b2 > bytes) bytes = b2;
  void* tmp = nullptr;
  CK(cudaMallocAsync(&tmp, bytes ? bytes : 16, s));
  CK(cub::DeviceSelect::Flagged(tmp, bytes, cub::CountingInputIterator<int>(0), flag, seg_node_dev,
                                counts_dev, n_nodes, s));
  k_seg_offsets<<<grid_for((long long)n_nodes + 1), 256, 0, s>>>(offsets_dev, seg_node_dev, counts_dev, n, seg_off_dev);
  k_tile_marks<<<grid_for(n_cand), 256, 0, s>>>(seg_off_dev, counts_dev, n_marks, tile, cand, flag);
  k_tile_flags<<<grid_for(n_cand), 256, 0, s>>>(cand, n_cand, flag);
  CK(cub::DeviceSelect::Flagged(tmp, bytes, cand, flag, tiles_dev, counts_dev + 1, n_cand, s));
  CK(cudaFreeAsync(tmp, s));
  CK(cudaFreeAsync(cand, s));
  CK(cudaFreeAsync(flag, s));
  CK(cudaGetLastError());
  return 0;
}

// gather/scatter of SoA arrays through a permutation (bind / download):
//   dst[k] = src[perm[k]]   (gather, to node-sorted order)
//   dst[perm[k]] = src[k]   (scatter back to instance order)
__global__ void k_permute(const double* __restrict__ src, double* __restrict__ dst,
                          const long long* __restrict__ perm, long long n, int inverse) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    long long j = perm[k];
    if (inverse)
      dst[j] = src[k];
    else
      dst[k] = src[j];
  }
}
NMODL_API int nmodl_permute(const double* src, double* dst, const long long* perm, long long n,
                            int inverse, cudaStream_t s) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  k_permute<<<blocks, 256, 0, s>>>(src, dst, perm, n, inverse);
  CK(cudaGetLastError());
  return 0;
}
__global__ void k_permute_i32(const int* __restrict__ src, int* __restrict__ dst,
                              const long long* __restrict__ perm, long long n) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x)
    dst[k] = src[perm[k]];
}
NMODL_API int nmodl_permute_i32(const int* src, int* dst, const long long* perm, long long n,
                                cudaStream_t s) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  k_permute_i32<<<blocks, 256, 0, s>>>(src, dst, perm, n);
  CK(cudaGetLastError());
  return 0;
}

// v[i] = node_v[node_index[i]]  (materialise per-instance voltage on download)
__global__ void k_gather_v(const double* __restrict__ node_v, const int* __restrict__ idx,
                           double* __restrict__ v, long long n) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x)
    v[k] = node_v[idx[k]];
}
NMODL_API int nmodl_gather_v(const double* node_v, const int* node_index, double* v, long long n,
                             cudaStream_t s) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  k_gather_v<<<blocks, 256, 0, s>>>(node_v, node_index, v, n);
  CK(cudaGetLastError());
  return 0;
}

// ---------------------------------------------------------------------------
// self-test: nmodl::exp_c against CUDA exp() on the same inputs
#include "nmodl_b200/mechanism.cuh"
__global__ void k_selftest_exp(const double* __restrict__ x, double* __restrict__ a, double* __restrict__ b,
                               long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    a[i] = nmodl::exp_c(x[i]);
    b[i] = exp(x[i]);
  }
}
NMODL_API int nmodl_selftest_exp(const double* x, double* a, double* b, long long n, cudaStream_t s) {
  k_selftest_exp<<<256, 256, 0, s>>>(x, a, b, n);
  CK(cudaGetLastError());
  return 0;
}
// relaxed division (CudaOptions.div_approx): out[i] = div_a(a[i], b[i]); the
// branch-free div_af must give the same value whenever it does not flag
__global__ void k_selftest_div_approx(const double* __restrict__ a, const double* __restrict__ b,
                                      double* __restrict__ out, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned f = 0;
    const double fast = nmodl::div_af(a[i], b[i], f);
    const double safe = nmodl::div_a(a[i], b[i]);
    out[i] = (f == 0 && __double_as_longlong(fast) != __double_as_longlong(safe)) ? __longlong_as_double(0x7ff4dead00000000ll) : safe;
  }
}
NMODL_API int nmodl_selftest_div_approx(const double* a, const double* b, double* out, long long n, cudaStream_t s) {
  k_selftest_div_approx<<<256, 256, 0, s>>>(a, b, out, n);
  CK(cudaGetLastError());
  return 0;
}

// shared-memory table exp (CudaOptions.exp_smem): out = exp16(x); flag bit 0 =
// fast form flagged, bit 1 = fast and safe forms disagree without a flag
__global__ void k_selftest_exp_smem(const double* __restrict__ x, double* __restrict__ a,
                                    unsigned* __restrict__ fl, long long n) {
  nmodl::exp16_init();
  __syncthreads();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned f = 0;
    const double fast = nmodl::exp16f(x[i], f);
    const double safe = nmodl::exp16(x[i]);
    a[i] = safe;
    fl[i] = f | ((f == 0 && __double_as_longlong(fast) != __double_as_longlong(safe)) ? 2u : 0u);
  }
}
NMODL_API int nmodl_selftest_exp_smem(const double* x, double* a, unsigned* fl, long long n, cudaStream_t s) {
  k_selftest_exp_smem<<<256, 256, 0, s>>>(x, a, fl, n);
  CK(cudaGetLastError());
  return 0;
}

// Deferred in-order fold of one-instance-per-node populations (seg_unique
// mode 2): the populations ran concurrently and left their currents in
// i_acc/g_acc; node k of instance j receives them in population order --
// the same operations, in the same order, as the sequential kernels' own
// node_rhs[nd] -= i / node_d[nd] += g.
struct nmodl_combine_args {
  const double* i[8];
  const double* g[8];
  int n_pops;
};
// P populations known at compile time: every population's i/g load of a
// node is in flight at once (a runtime-bounded loop issued them one L2
// round trip after another: 5 populations took ~2 us at 12.5k nodes); the
// arithmetic is the same chain in the same order.  PDL (flags bit 0): the
// grid is launched for programmatic dependent launch behind the kernel
// before it on the stream, loads the population currents (complete: they
// come from full dependencies, e.g. another stream's kernel joined by an
// event) and waits for that kernel only before it touches node rhs/d --
// the caller vouches that the predecessor writes no i/g array it reads.
template <int P, bool PDL>
__global__ void k_combine_unique(double* __restrict__ rhs, double* __restrict__ d, const int* __restrict__ node_index,
                                 long long n, const nmodl_combine_args a) {
  // a following kernel launched for programmatic dependent launch (the
  // synapse step, CudaOptions.pdl) may be scheduled now; it waits for this
  // grid's completion before it reads anything
  asm volatile("griddepcontrol.launch_dependents;");
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (PDL) {
    // one node per thread (the launch covers n): loads before the wait
    double iv[P], gv[P];
    int nd = 0;
    if (j < n) {
#pragma unroll
      for (int p = 0; p < P; ++p) {
        iv[p] = __ldcg(a.i[p] + j);
        gv[p] = __ldcg(a.g[p] + j);
      }
      nd = node_index[j];
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (j < n) {
      double r = rhs[nd], dd = d[nd];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        r = r - iv[p];
        dd = dd + gv[p];
      }
      rhs[nd] = r;
      d[nd] = dd;
    }
    return;
  }
  for (; j < n; j += stride) {
    double iv[P], gv[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      iv[p] = __ldcg(a.i[p] + j);
      gv[p] = __ldcg(a.g[p] + j);
    }
    const int nd = node_index[j];
    double r = rhs[nd], dd = d[nd];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      r = r - iv[p];
      dd = dd + gv[p];
    }
    rhs[nd] = r;
    d[nd] = dd;
  }
}
NMODL_API int nmodl_combine_unique_ex(double* rhs, double* d, const int* node_index, long long n,
                                      const double* const* i_ptrs, const double* const* g_ptrs, int n_pops, int flags,
                                      cudaStream_t s) {
  if (n_pops < 0 || n_pops > 8) return (int)cudaErrorInvalidValue;
  if (n <= 0 || n_pops == 0) return 0;  // nothing to fold
  nmodl_combine_args a{};
  for (int p = 0; p < n_pops; ++p) {
    a.i[p] = i_ptrs[p];
    a.g[p] = g_ptrs[p];
  }
  a.n_pops = n_pops;
  const long long blocks = (n + 255) / 256;
  const bool pdl = (flags & 1) != 0;
  if (pdl && blocks > (1LL << 30)) return (int)cudaErrorInvalidValue;
  const int grid = pdl ? (int)blocks : (int)(blocks < 148 * 16 ? blocks : 148 * 16);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  switch (n_pops) {
#define NM_COMBINE(P)                                                                                          \
  case P:                                                                                                      \
    if (pdl) CK(cudaLaunchKernelEx(&cfg, k_combine_unique<P, true>, rhs, d, node_index, n, a));                \
    else CK(cudaLaunchKernelEx(&cfg, k_combine_unique<P, false>, rhs, d, node_index, n, a));                   \
    break;
    NM_COMBINE(1) NM_COMBINE(2) NM_COMBINE(3) NM_COMBINE(4) NM_COMBINE(5) NM_COMBINE(6) NM_COMBINE(7)
    NM_COMBINE(8)
#undef NM_COMBINE
  }
  CK(cudaGetLastError());
  return 0;
}
NMODL_API int nmodl_combine_unique(double* rhs, double* d, const int* node_index, long long n,
                                   const double* const* i_ptrs, const double* const* g_ptrs, int n_pops,
                                   cudaStream_t s) {
  return nmodl_combine_unique_ex(rhs, d, node_index, n, i_ptrs, g_ptrs, n_pops, 0, s);
}



// ---------------------------------------------------------------------------
// NCCL (validation collectives only: the hot path has no exchange).  The
// library is opened at first use (libnccl.so.2 of the image), so the runtime
// loads on hosts without NCCL and a multi-GPU call fails loudly there.
// Bootstrap of the unique id is the caller's (parallel.py: a file shared by
// the ranks of one node).
#include <dlfcn.h>
#include <nccl.h>

namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;

int nccl_load() {
  if (g_nccl.h) return 0;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
  if (!h) {
    snprintf(g_err, sizeof(g_err), "NCCL not available: %s", dlerror());
    return 1000;
  }
  g_nccl.get_unique_id = (decltype(g_nccl.get_unique_id))dlsym(h, "ncclGetUniqueId");
  g_nccl.comm_init_rank = (decltype(g_nccl.comm_init_rank))dlsym(h, "ncclCommInitRank");
  g_nccl.comm_destroy = (decltype(g_nccl.comm_destroy))dlsym(h, "ncclCommDestroy");
  g_nccl.all_reduce = (decltype(g_nccl.all_reduce))dlsym(h, "ncclAllReduce");
  g_nccl.all_gather = (decltype(g_nccl.all_gather))dlsym(h, "ncclAllGather");
  g_nccl.error_string = (decltype(g_nccl.error_string))dlsym(h, "ncclGetErrorString");
  if (!g_nccl.get_unique_id || !g_nccl.comm_init_rank || !g_nccl.comm_destroy || !g_nccl.all_reduce ||
      !g_nccl.all_gather || !g_nccl.error_string) {
    snprintf(g_err, sizeof(g_err), "NCCL symbols missing in the loaded library");
    return 1001;
  }
  g_nccl.h = h;
  return 0;
}

int nccl_fail(ncclResult_t r, const char* what) {
  snprintf(g_err, sizeof(g_err), "%s: NCCL error %d (%s)", what, (int)r,
           g_nccl.error_string ? g_nccl.error_string(r) : "?");
  return 2000 + (int)r;
}
}  // namespace

#define NCK(call, what)                               \
  do {                                                \
    ncclResult_t r_ = (call);                         \
    if (r_ != ncclSuccess) return nccl_fail(r_, what); \
  } while (0)

NMODL_API int nmodl_nccl_unique_id(unsigned char* out128) {
  if (int rc = nccl_load()) return rc;
  ncclUniqueId id;
  NCK(g_nccl.get_unique_id(&id), "ncclGetUniqueId");
  memcpy(out128, id.internal, NCCL_UNIQUE_ID_BYTES);
  return 0;
}
NMODL_API int nmodl_nccl_init(void** comm, int nranks, const unsigned char* id128, int rank) {
  if (int rc = nccl_load()) return rc;
  ncclUniqueId id;
  memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t c = nullptr;
  NCK(g_nccl.comm_init_rank(&c, nranks, id, rank), "ncclCommInitRank");
  *comm = (void*)c;
  return 0;
}
NMODL_API int nmodl_nccl_destroy(void* comm) {
  if (int rc = nccl_load()) return rc;
  NCK(g_nccl.comm_destroy((ncclComm_t)comm), "ncclCommDestroy");
  return 0;
}
// op: 0 sum, 1 max (fp64)
NMODL_API int nmodl_nccl_allreduce_f64(void* comm, const double* send, double* recv, long long count, int op,
                                       cudaStream_t s) {
  if (int rc = nccl_load()) return rc;
  NCK(g_nccl.all_reduce(send, recv, (size_t)count, ncclFloat64, op == 1 ? ncclMax : ncclSum, (ncclComm_t)comm, s),
      "ncclAllReduce");
  return 0;
}
NMODL_API int nmodl_nccl_allgather_f64(void* comm, const double* send, double* recv, long long count, cudaStream_t s) {
  if (int rc = nccl_load()) return rc;
  NCK(g_nccl.all_gather(send, recv, (size_t)count, ncclFloat64, (ncclComm_t)comm, s), "ncclAllGather");
  return 0;
}
