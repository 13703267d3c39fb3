// C-ABI of libparse (include/parse.h): validation, schedule upload, TMA
// descriptor encoding and kernel launch.  No compute happens here; every step
// of the path runs in the kernels.  There is no fallback path: a device other
// than sm_100 is PARSE_ERR_UNSUPPORTED.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include <cudaTypedefs.h>

#include "internal.h"

namespace parse {
namespace {

thread_local std::string g_err;

parse_status_t fail(parse_status_t s, const std::string& msg) {
  g_err = msg;
  return s;
}
parse_status_t cuda_fail(cudaError_t e, const char* what) {
  return fail(PARSE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct DeviceInfo { int major = -1, minor = -1, sms = 0; };

parse_status_t check_device(DeviceInfo* out) {
  static std::mutex mu;
  static DeviceInfo cache[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (dev < 0 || dev >= 64) return fail(PARSE_ERR_UNSUPPORTED, "device index out of range");
  std::lock_guard<std::mutex> lk(mu);
  DeviceInfo& di = cache[dev];
  if (di.major < 0) {
    if ((e = cudaDeviceGetAttribute(&di.major, cudaDevAttrComputeCapabilityMajor, dev)) != cudaSuccess ||
        (e = cudaDeviceGetAttribute(&di.minor, cudaDevAttrComputeCapabilityMinor, dev)) != cudaSuccess ||
        (e = cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) {
      di.major = -1;
      return cuda_fail(e, "cudaDeviceGetAttribute");
    }
  }
  if (di.major != 10 || di.minor != 0)
    return fail(PARSE_ERR_UNSUPPORTED, "libparse is built for sm_100a (B200); device is sm_" +
                                           std::to_string(di.major) + std::to_string(di.minor));
  *out = di;
  return PARSE_OK;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// 4-D map over [B][L][H][D] (D contiguous) of bf16 (elem = 2) or e4m3 (elem =
// 1, moved as bytes), box {128 B of d, box_h, box_t, 1}, 128-byte swizzle
// (matches the UMMA K-major / MN-major SW128 layouts).
parse_status_t make_map(CUtensorMap* m, const void* base, int D, int H, int64_t L, int64_t B,
                        const int64_t strides[3], int box_h, int box_t, int elem = 2) {
  auto enc = get_encode();
  if (!enc) return fail(PARSE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {cuuint64_t(D), cuuint64_t(H), cuuint64_t(L), cuuint64_t(B)};
  cuuint64_t gstr[3] = {cuuint64_t(strides[2]) * elem, cuuint64_t(strides[1]) * elem, cuuint64_t(strides[0]) * elem};
  cuuint32_t box[4] = {cuuint32_t(128 / elem), cuuint32_t(box_h), cuuint32_t(box_t), 1u};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, elem == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 4,
                   const_cast<void*>(base), dims, gstr, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PARSE_ERR_INVALID, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) +
                                                            "): check strides/alignment");
  return PARSE_OK;
}

// ---------------------------------------------------------------------------
// Schedule images.  The workspace content of a problem (zeroed work counter,
// request table, boundaries, tree masks, work items) is built once on the host
// into a pinned, device-mapped buffer and cached by the exact problem
// (per device, LRU), with a device-resident copy filled once by the copy
// engine.  Every call copies the device image into the caller's workspace with
// upload_kernel (HBM to HBM, ~1 us for config 3's 1.3 MB): no host rebuild per
// call, and no per-call copy-engine transfer that would queue behind a serving
// loop's bulk input copies.  (Round 2's first form read the mapped pinned
// image over PCIe in every call: ~0.25 ms per call on config 3, latency-bound;
// DESIGN §8.)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) upload_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                    int64_t n16) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  // up to four independent 16-byte loads in flight per thread
  for (; i + 3 * stride < n16; i += 4 * stride) {
    const uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
  }
  for (; i < n16; i += stride) dst[i] = src[i];
}

struct Prepared {
  WorkspaceLayout wl{};
  size_t n_items = 0, n_pairs = 0;
};

struct SchedImage {
  std::vector<int64_t> key;     // exact serialisation of the problem (no hash collisions)
  int device = -1;
  void* host = nullptr;         // pinned staging copy; wl.total bytes
  void* dev = nullptr;          // device-resident copy on `device` (the upload source)
  Prepared prep;
  cudaEvent_t last_use = nullptr;
  uint64_t tick = 0;
};

constexpr size_t kImageCacheEntries = 16;
constexpr size_t kImageCacheBytes = size_t(256) << 20;
std::mutex g_img_mu;
std::vector<SchedImage*> g_images;
uint64_t g_img_tick = 0;

std::vector<int64_t> problem_key(const Problem& p, bool bf16, int device) {
  std::vector<int64_t> k = {device, bf16, p.B, p.Hq, p.Hkv, p.D, p.S, p.N, p.K, p.L, p.varlen, p.self_align,
                            p.tree, int64_t(p.bnd.size())};
  auto add = [&](const std::vector<int32_t>& v) { k.insert(k.end(), v.begin(), v.end()); };
  add(p.Nb); add(p.Kb); add(p.bnd_off); add(p.bnd); add(p.q_row0); add(p.kv_row0);
  for (uint64_t a : p.anc) k.push_back(int64_t(a));
  return k;
}

void free_image(SchedImage* im) {
  if (im->last_use) {
    cudaEventSynchronize(im->last_use);   // its last upload has read the buffers
    cudaEventDestroy(im->last_use);
  }
  if (im->dev) {
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != im->device) cudaSetDevice(im->device);
    cudaFree(im->dev);
    if (cur != im->device && cur >= 0) cudaSetDevice(cur);
  }
  if (im->host) cudaFreeHost(im->host);
  delete im;
}

// Fill the host image of problem p (layout wl).
void fill_image(const Problem& p, const WorkspaceLayout& wl, const std::vector<WorkItem>& items,
                const std::vector<int2>& pairs, uint8_t* h) {
  std::memset(h, 0, wl.total);
  ReqDesc* rd = reinterpret_cast<ReqDesc*>(h + wl.req_off);
  for (int b = 0; b < p.B; ++b)
    rd[b] = ReqDesc{p.Nb[b], p.Lb(b), p.Kb[b], p.bnd_off[b], p.q_row0[b], p.kv_row0[b], p.varlen ? 0 : b, 0};
  if (!p.bnd.empty()) std::memcpy(h + wl.bnd_off, p.bnd.data(), sizeof(int32_t) * p.bnd.size());
  if (p.tree) std::memcpy(h + wl.anc_off, p.anc.data(), sizeof(uint64_t) * p.anc.size());
  if (!items.empty()) std::memcpy(h + wl.items_off, items.data(), sizeof(WorkItem) * items.size());
  if (!pairs.empty()) std::memcpy(h + wl.pairs_off, pairs.data(), sizeof(int2) * pairs.size());
}

// Look up (or build) the image of p and enqueue its copy into `workspace`.
parse_status_t upload_schedule(const Problem& p, bool bf16, int device, void* workspace, size_t workspace_bytes,
                               cudaStream_t stream, Prepared* out) {
  std::vector<int64_t> key = problem_key(p, bf16, device);
  std::lock_guard<std::mutex> lk(g_img_mu);
  SchedImage* im = nullptr;
  for (SchedImage* e : g_images)
    if (e->key == key) { im = e; break; }
  cudaError_t e;
  if (!im) {
    std::unique_ptr<SchedImage> ni(new SchedImage);
    ni->key = std::move(key);
    ni->device = device;
    ni->prep.wl = workspace_layout(p, bf16);
    std::vector<WorkItem> items;
    std::vector<int2> pairs;
    if (bf16) build_schedule(p, &items);
#ifdef PARSE_WITH_2SM
    if (bf16) build_pairs(items, p.Hkv, p.Hq, &pairs);
#else
    if (bf16) build_units(items, p.Hkv, p.Hq, &pairs);   // the 2-CTA cluster kernel's work list
#endif
    ni->prep.n_items = items.size();
    ni->prep.n_pairs = pairs.size();
    if ((e = cudaHostAlloc(&ni->host, ni->prep.wl.total, cudaHostAllocPortable)) != cudaSuccess) {
      ni->host = nullptr;
      return cuda_fail(e, "cudaHostAlloc (schedule image)");
    }
    fill_image(p, ni->prep.wl, items, pairs, static_cast<uint8_t*>(ni->host));
    if ((e = cudaMalloc(&ni->dev, ni->prep.wl.total)) != cudaSuccess) {
      ni->dev = nullptr;
      cudaFreeHost(ni->host);
      return cuda_fail(e, "cudaMalloc (schedule image)");
    }
    if ((e = cudaEventCreateWithFlags(&ni->last_use, cudaEventDisableTiming)) != cudaSuccess) {
      cudaFree(ni->dev);
      cudaFreeHost(ni->host);
      return cuda_fail(e, "cudaEventCreate");
    }
    // once per image: the copy engine fills the device copy (stream-ordered
    // before this call's upload_kernel; last_use, recorded below, covers it)
    if ((e = cudaMemcpyAsync(ni->dev, ni->host, ni->prep.wl.total, cudaMemcpyHostToDevice, stream)) != cudaSuccess) {
      cudaEventDestroy(ni->last_use);
      cudaFree(ni->dev);
      cudaFreeHost(ni->host);
      return cuda_fail(e, "cudaMemcpyAsync (schedule image)");
    }
    // LRU eviction by entry count and pinned bytes
    size_t bytes = ni->prep.wl.total;
    for (SchedImage* x : g_images) bytes += x->prep.wl.total;
    while (!g_images.empty() && (g_images.size() >= kImageCacheEntries || bytes > kImageCacheBytes)) {
      auto lru = std::min_element(g_images.begin(), g_images.end(),
                                  [](const SchedImage* a, const SchedImage* b) { return a->tick < b->tick; });
      bytes -= (*lru)->prep.wl.total;
      free_image(*lru);
      g_images.erase(lru);
    }
    im = ni.release();
    g_images.push_back(im);
  }
  im->tick = ++g_img_tick;
  if (!workspace || workspace_bytes < im->prep.wl.total)
    return fail(PARSE_ERR_WORKSPACE, "workspace needs " + std::to_string(im->prep.wl.total) + " bytes");
  const int64_t n16 = int64_t(im->prep.wl.total / 16);   // total is 256-byte aligned
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(4 * 148, (n16 + 255) / 256)));
  upload_kernel<<<blocks, 256, 0, stream>>>(static_cast<const uint4*>(im->dev), static_cast<uint4*>(workspace),
                                            n16);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "upload_kernel launch");
  if ((e = cudaEventRecord(im->last_use, stream)) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
  *out = im->prep;
  return PARSE_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Geometry of one of Q/K/V as a 4-D TMA map (d, head, row, outer): `rows`
// rows per outer index; strides (outer, row, head) in elements.
struct Geom { int64_t rows, outer; int64_t strides[3]; };

struct VerifyIO {
  const void *q, *k, *v;
  void* o;
  float* lse;
  Geom q_geom, k_geom, v_geom;
  int64_t o_strides[3];        // (outer, row, head)
  int64_t lse_sb, lse_sh;
  int32_t page_log2, num_pages, bt_stride;   // paged K/V (page_log2 > 0)
  const int32_t* block_table;
  float descale[3] = {1.f, 1.f, 1.f};         // FP8: Q, K, V descale factors
};

// Validation + schedule upload into the workspace (zeroes the work counter).
parse_status_t prepare_verify(const Problem& p, int precision, void* workspace, size_t workspace_bytes,
                              cudaStream_t stream, Prepared* out) {
  if (precision != PARSE_PREC_BF16 && precision != PARSE_PREC_FP32_DEBUG && precision != PARSE_PREC_FP8_E4M3)
    return fail(PARSE_ERR_INVALID, "unknown precision");
  const bool fp8 = precision == PARSE_PREC_FP8_E4M3;
  if (fp8 && p.D != 128) return fail(PARSE_ERR_UNSUPPORTED, "FP8 path: head_dim 128 only");
  parse_status_t s;
  DeviceInfo di;
  if ((s = check_device(&di)) != PARSE_OK) return s;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  const bool bf16 = precision != PARSE_PREC_FP32_DEBUG;   // tcgen05 path (bf16 or FP8)
  return upload_schedule(p, bf16, dev, workspace, workspace_bytes, stream, out);
}

// Tensor maps + launch over a prepared workspace.  Only host-side encoding,
// (optionally) a memset of the work counter and the kernel launch: capturable
// into a CUDA graph.
parse_status_t launch_prepared(const Problem& p, int precision, const VerifyIO& io, void* workspace,
                               const Prepared& prep, bool reset_counter, cudaStream_t stream) {
  if (!io.q || !io.k || !io.v || !io.o) return fail(PARSE_ERR_INVALID, "q, k, v, o must be non-NULL device pointers");
  if (!aligned16(io.q) || !aligned16(io.k) || !aligned16(io.v) || !aligned16(io.o) || (io.lse && !aligned16(io.lse)))
    return fail(PARSE_ERR_INVALID, "q, k, v, o, lse must be 16-byte aligned");
  parse_status_t s;
  DeviceInfo di;
  if ((s = check_device(&di)) != PARSE_OK) return s;
  const bool fp8 = precision == PARSE_PREC_FP8_E4M3;
  const bool bf16 = precision != PARSE_PREC_FP32_DEBUG;
  const WorkspaceLayout& wl = prep.wl;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  if (reset_counter && bf16) {
    cudaError_t e = cudaMemsetAsync(ws + wl.counter_off, 0, sizeof(int32_t), stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  }
  const ReqDesc* d_req = reinterpret_cast<const ReqDesc*>(ws + wl.req_off);
  const int32_t* d_bnd = reinterpret_cast<const int32_t*>(ws + wl.bnd_off);
  const uint64_t* d_anc = p.tree ? reinterpret_cast<const uint64_t*>(ws + wl.anc_off) : nullptr;
  cudaError_t e;
  if (bf16) {
    CUtensorMap tq, tqp, tk, tv;
    const int hpt_s = suffix_heads_per_tile(p);
    // 2-CTA clusters with K/V multicast (dense, packed-row and paged K/V)
#if !defined(PARSE_NO_CLUSTER) && !defined(PARSE_WITH_PAIR) && !defined(PARSE_WITH_2SM)
    const bool cluster = true;
#else
    const bool cluster = false;   // A/B and experimental-kernel builds: the one-CTA kernel's maps
#endif
    const int kv_box = io.page_log2 ? std::min(1 << io.page_log2, kTile) : kTile;
    auto map = [&](CUtensorMap* m, const void* base, int H, const Geom& g, int box_h, int box_t) {
      return make_map(m, base, p.D, H, g.rows, g.outer, g.strides, box_h, box_t, fp8 ? 1 : 2);
    };
    if ((s = map(&tq, io.q, p.Hq, io.q_geom, 1, kTile)) != PARSE_OK) return s;
    if (hpt_s) {
      if ((s = map(&tqp, io.q, p.Hq, io.q_geom, hpt_s, p.S)) != PARSE_OK) return s;
    } else {
      tqp = tq;
    }
    if ((s = map(&tk, io.k, p.Hkv, io.k_geom, 1, kv_box)) != PARSE_OK) return s;
    if ((s = map(&tv, io.v, p.Hkv, io.v_geom, 1, kv_box)) != PARSE_OK) return s;
    AttnParams prm{};
    prm.req = d_req;
    prm.bnd = d_bnd;
    prm.anc = d_anc;
    prm.items = reinterpret_cast<const WorkItem*>(ws + wl.items_off);
    prm.n_items = int32_t(prep.n_items);
    prm.work = reinterpret_cast<const int2*>(ws + wl.pairs_off);
    prm.n_work = int32_t(prep.n_pairs);
    prm.counter = reinterpret_cast<int32_t*>(ws + wl.counter_off);
    prm.B = p.B; prm.Hq = p.Hq; prm.Hkv = p.Hkv; prm.S = p.S;
    if (!p.varlen) { prm.dense_N = p.N; prm.dense_K = p.K; prm.dense_L = p.L; }
    prm.scale_log2 = p.scale * 1.4426950408889634f * io.descale[0] * io.descale[1];
    prm.o_scale = io.descale[2];
    prm.page_log2 = io.page_log2; prm.num_pages = io.num_pages; prm.bt_stride = io.bt_stride;
    prm.block_table = io.block_table;
    prm.o = io.o;
    prm.lse = io.lse;
    prm.lse_sb = io.lse_sb; prm.lse_sh = io.lse_sh;
    prm.o_s0 = io.o_strides[0]; prm.o_s1 = io.o_strides[1]; prm.o_s2 = io.o_strides[2];
    // bf16 O: 32-byte alignment of the base and of every stride (16 elements)
    prm.o_v8 = (reinterpret_cast<uintptr_t>(io.o) % 32 == 0) && io.o_strides[0] % 16 == 0 &&
               io.o_strides[1] % 16 == 0 && io.o_strides[2] % 16 == 0;
    prm.trace = nullptr;
#if defined(PARSE_TRACE) || defined(PARSE_CTASTAT)
    if (const char* tp = std::getenv("PARSE_TRACE_PTR")) prm.trace = reinterpret_cast<long long*>(std::strtoull(tp, nullptr, 10));
#endif
#ifdef PARSE_WITH_PAIR
    // experimental build variant only (libparse_pair.so): the
    // CTA-pair kernel (S and P double-buffered in TMEM) for bf16 head_dim 128
    // with dense or packed-row K/V; measured slower than the one-CTA kernel.
    if (!fp8 && p.D == 128 && !io.page_log2) {
      CUtensorMap tk64;
      if ((s = make_map(&tk64, io.k, p.D, p.Hkv, io.k_geom.rows, io.k_geom.outer, io.k_geom.strides, 1, 64, 2)) !=
          PARSE_OK)
        return s;
      if ((e = launch_attn_pair(prm, tq, tqp, tk64, tv, di.sms, stream)) != cudaSuccess)
        return cuda_fail(e, "attn_pair launch");
    } else
#endif
#ifdef PARSE_WITH_2SM
    // experimental build variant only (libparse_2sm.so): the
    // cta_group::2 kernel for bf16 head_dim 128 dense / packed-row K/V.  The
    // default libparse.so has one attention kernel family and no switch.
    if (!fp8 && p.D == 128 && !io.page_log2) {
      CUtensorMap tk64;
      if ((s = make_map(&tk64, io.k, p.D, p.Hkv, io.k_geom.rows, io.k_geom.outer, io.k_geom.strides, 1, 64, 2)) !=
          PARSE_OK)
        return s;
      if ((e = launch_attn_sm100_2sm(prm, tq, tqp, tk64, tv, di.sms, stream)) != cudaSuccess)
        return cuda_fail(e, "attn_sm100_2sm launch");
    } else
#endif
    {
      if ((e = launch_attn_sm100(prm, p.D, fp8, cluster, tq, tqp, tk, tv, di.sms, stream)) != cudaSuccess)
        return cuda_fail(e, "attn_sm100 launch");
    }
  } else {
    AttnFp32Params prm{};
    prm.q = static_cast<const uint16_t*>(io.q);
    prm.k = static_cast<const uint16_t*>(io.k);
    prm.v = static_cast<const uint16_t*>(io.v);
    prm.o = static_cast<float*>(io.o);
    prm.lse = io.lse;
    prm.req = d_req;
    prm.bnd = d_bnd;
    prm.anc = d_anc;
    prm.B = p.B; prm.Hq = p.Hq; prm.Hkv = p.Hkv; prm.D = p.D; prm.S = p.S; prm.Lmax = p.L;
    prm.scale = p.scale;
    prm.page_log2 = io.page_log2; prm.num_pages = io.num_pages; prm.bt_stride = io.bt_stride;
    prm.block_table = io.block_table;
    prm.lse_sb = io.lse_sb; prm.lse_sh = io.lse_sh;
    prm.q_s0 = io.q_geom.strides[0]; prm.q_s1 = io.q_geom.strides[1]; prm.q_s2 = io.q_geom.strides[2];
    prm.k_s0 = io.k_geom.strides[0]; prm.k_s1 = io.k_geom.strides[1]; prm.k_s2 = io.k_geom.strides[2];
    prm.v_s0 = io.v_geom.strides[0]; prm.v_s1 = io.v_geom.strides[1]; prm.v_s2 = io.v_geom.strides[2];
    prm.o_s0 = io.o_strides[0]; prm.o_s1 = io.o_strides[1]; prm.o_s2 = io.o_strides[2];
    if ((e = launch_attn_fp32(prm, stream)) != cudaSuccess) return cuda_fail(e, "attn_fp32 launch");
  }
  g_err.clear();
  return PARSE_OK;
}

parse_status_t launch_verify(const Problem& p, int precision, const VerifyIO& io, void* workspace,
                             size_t workspace_bytes, cudaStream_t stream) {
  if (!io.q || !io.k || !io.v || !io.o) return fail(PARSE_ERR_INVALID, "q, k, v, o must be non-NULL device pointers");
  Prepared prep;
  parse_status_t s = prepare_verify(p, precision, workspace, workspace_bytes, stream, &prep);
  if (s != PARSE_OK) return s;
  return launch_prepared(p, precision, io, workspace, prep, false, stream);
}

double logit_threshold(double tau) {
  if (tau <= 0.0) return -INFINITY;
  if (tau >= 1.0) return INFINITY;
  return std::log(tau) - std::log1p(-tau);
}

}  // namespace
}  // namespace parse

using namespace parse;

extern "C" {

const char* parse_last_error(void) { return g_err.c_str(); }

int parse_version(void) { return PARSE_VERSION; }

parse_status_t parse_suffix_positions(const int32_t* boundaries, int32_t K, int32_t S, int32_t* positions) {
  if (!boundaries || !positions || K < 1 || S < 1) return fail(PARSE_ERR_INVALID, "bad arguments");
  for (int k = 0; k < K; ++k)
    for (int s = 0; s < S; ++s) positions[int64_t(k) * S + s] = boundaries[k] + s;
  g_err.clear();
  return PARSE_OK;
}

parse_status_t parse_verify_attn_workspace_size(const parse_attn_desc_t* desc, size_t* bytes) {
  Problem p;
  std::string err;
  parse_status_t s = make_problem(desc, &p, &err);
  if (s != PARSE_OK) return fail(s, err);
  if (!bytes) return fail(PARSE_ERR_INVALID, "bytes is NULL");
  *bytes = workspace_layout(p, desc->precision != PARSE_PREC_FP32_DEBUG).total;
  g_err.clear();
  return PARSE_OK;
}

parse_status_t parse_verify_attn_schedule(const parse_attn_desc_t* desc, parse_work_item_t* out, size_t capacity,
                                          size_t* n_items) {
  static_assert(sizeof(parse_work_item_t) == sizeof(WorkItem), "public and internal work items match");
  Problem p;
  std::string err;
  parse_status_t s = make_problem(desc, &p, &err);
  if (s != PARSE_OK) return fail(s, err);
  if (!n_items) return fail(PARSE_ERR_INVALID, "n_items is NULL");
  std::vector<WorkItem> items;
  build_schedule(p, &items);
  *n_items = items.size();
  if (out) std::memcpy(out, items.data(), sizeof(WorkItem) * std::min(capacity, items.size()));
  g_err.clear();
  return PARSE_OK;
}

parse_status_t parse_verify_attn_units(const parse_attn_desc_t* desc, int32_t* out, size_t capacity,
                                       size_t* n_units) {
  Problem p;
  std::string err;
  parse_status_t s = make_problem(desc, &p, &err);
  if (s != PARSE_OK) return fail(s, err);
  if (!n_units) return fail(PARSE_ERR_INVALID, "n_units is NULL");
  std::vector<WorkItem> items;
  build_schedule(p, &items);
  std::vector<int2> units;
  build_units(items, p.Hkv, p.Hq, &units);
  *n_units = units.size();
  if (out) std::memcpy(out, units.data(), sizeof(int2) * std::min(capacity, units.size()));
  g_err.clear();
  return PARSE_OK;
}

parse_status_t parse_verify_attn(const parse_attn_desc_t* desc, const void* q, const void* k, const void* v,
                                 void* o, float* lse, void* workspace, size_t workspace_bytes, void* stream_) {
  Problem p;
  std::string err;
  parse_status_t s = make_problem(desc, &p, &err);
  if (s != PARSE_OK) return fail(s, err);
  // dense BSHD: TMA dims (d, head, row, batch), strides (batch, row, head)
  VerifyIO io{};
  io.q = q; io.k = k; io.v = v; io.o = o; io.lse = lse;
  io.q_geom = {p.L, p.B, {desc->q_strides[0], desc->q_strides[1], desc->q_strides[2]}};
  io.k_geom = {p.L, p.B, {desc->k_strides[0], desc->k_strides[1], desc->k_strides[2]}};
  io.v_geom = {p.L, p.B, {desc->v_strides[0], desc->v_strides[1], desc->v_strides[2]}};
  for (int i = 0; i < 3; ++i) io.o_strides[i] = desc->o_strides[i];
  io.lse_sb = int64_t(p.Hq) * p.L;
  io.lse_sh = p.L;
  if (desc->precision == PARSE_PREC_FP8_E4M3)
    return fail(PARSE_ERR_INVALID, "PARSE_PREC_FP8_E4M3 inputs go through parse_verify_attn_fp8");
  return launch_verify(p, desc->precision, io, workspace, workspace_bytes, static_cast<cudaStream_t>(stream_));
}

// ---------------------------------------------------------------------------
// Plans: schedule built and uploaded once, launches capturable into CUDA graphs
// ---------------------------------------------------------------------------
struct parse_attn_plan_s {
  Problem p;
  int precision;
  VerifyIO io;          // geometry only; pointers are per run
  void* workspace;
  Prepared prep;
};

parse_status_t parse_verify_attn_plan_create(const parse_attn_desc_t* desc, void* workspace, size_t workspace_bytes,
                                             void* stream_, parse_attn_plan_t* plan) {
  if (!plan) return fail(PARSE_ERR_INVALID, "plan is NULL");
  *plan = nullptr;
  Problem p;
  std::string err;
  parse_status_t s = make_problem(desc, &p, &err);
  if (s != PARSE_OK) return fail(s, err);
  if (desc->precision != PARSE_PREC_BF16 && desc->precision != PARSE_PREC_FP32_DEBUG)
    return fail(PARSE_ERR_UNSUPPORTED, "plans support PARSE_PREC_BF16 and PARSE_PREC_FP32_DEBUG");
  VerifyIO io{};
  io.q_geom = {p.L, p.B, {desc->q_strides[0], desc->q_strides[1], desc->q_strides[2]}};
  io.k_geom = {p.L, p.B, {desc->k_strides[0], desc->k_strides[1], desc->k_strides[2]}};
  io.v_geom = {p.L, p.B, {desc->v_strides[0], desc->v_strides[1], desc->v_strides[2]}};
  for (int i = 0; i < 3; ++i) io.o_strides[i] = desc->o_strides[i];
  io.lse_sb = int64_t(p.Hq) * p.L;
  io.lse_sh = p.L;
  Prepared prep;
  s = prepare_verify(p, desc->precision, workspace, workspace_bytes, static_cast<cudaStream_t>(stream_), &prep);
  if (s != PARSE_OK) return s;
  *plan = new parse_attn_plan_s{p, desc->precision, io, workspace, prep};
  g_err.clear();
  return PARSE_OK;
}

parse_status_t parse_verify_attn_plan_run(parse_attn_plan_t plan, const void* q, const void* k, const void* v, void* o,
                                          float* lse, void* stream_) {
  if (!plan) return fail(PARSE_ERR_INVALID, "plan is NULL");
  VerifyIO io = plan->io;
  io.q = q; io.k = k; io.v = v; io.o = o; io.lse = lse;
  return launch_prepared(plan->p, plan->precision, io, plan->workspace, plan->prep, true,
                         static_cast<cudaStream_t>(stream_));
}

parse_status_t parse_verify_attn_plan_destroy(parse_attn_plan_t plan) {
  delete plan;
  g_err.clear();
  return PARSE_OK;
}

parse_status_t parse_verify_attn_fp8(const parse_attn_desc_t* desc, const void* q, const void* k, const void* v,
                                     float descale_q, float descale_k, float descale_v, void* o, float* lse,
                                     void* workspace, size_t workspace_bytes, void* stream_) {
  Problem p;
  std::string err;
  parse_status_t s = make_problem(desc, &p, &err);
  if (s != PARSE_OK) return fail(s, err);
  if (desc->precision != PARSE_PREC_FP8_E4M3) return fail(PARSE_ERR_INVALID, "desc->precision must be PARSE_PREC_FP8_E4M3");
  const int64_t* st[3] = {desc->q_strides, desc->k_strides, desc->v_strides};
  for (int t = 0; t < 3; ++t)
    for (int i = 0; i < 3; ++i)
      if (st[t][i] % 16) return fail(PARSE_ERR_INVALID, "FP8 q/k/v strides must be multiples of 16 elements");
  if (!(descale_q > 0.f) || !(descale_k > 0.f) || !(descale_v > 0.f) || !std::isfinite(descale_q) ||
      !std::isfinite(descale_k) || !std::isfinite(descale_v))
    return fail(PARSE_ERR_INVALID, "descale factors must be positive and finite");
  VerifyIO io{};
  io.q = q; io.k = k; io.v = v; io.o = o; io.lse = lse;
  io.q_geom = {p.L, p.B, {desc->q_strides[0], desc->q_strides[1], desc->q_strides[2]}};
  io.k_geom = {p.L, p.B, {desc->k_strides[0], desc->k_strides[1], desc->k_strides[2]}};
  io.v_geom = {p.L, p.B, {desc->v_strides[0], desc->v_strides[1], desc->v_strides[2]}};
  for (int i = 0; i < 3; ++i) io.o_strides[i] = desc->o_strides[i];
  io.lse_sb = int64_t(p.Hq) * p.L;
  io.lse_sh = p.L;
  io.descale[0] = descale_q; io.descale[1] = descale_k; io.descale[2] = descale_v;
  return launch_verify(p, PARSE_PREC_FP8_E4M3, io, workspace, workspace_bytes, static_cast<cudaStream_t>(stream_));
}

parse_status_t parse_verify_attn_varlen_workspace_size(const parse_varlen_desc_t* desc, size_t* bytes) {
  Problem p;
  std::string err;
  parse_status_t s = make_problem_varlen(desc, &p, &err);
  if (s != PARSE_OK) return fail(s, err);
  if (!bytes) return fail(PARSE_ERR_INVALID, "bytes is NULL");
  *bytes = workspace_layout(p, desc->precision != PARSE_PREC_FP32_DEBUG).total;
  g_err.clear();
  return PARSE_OK;
}

parse_status_t parse_verify_attn_varlen_schedule(const parse_varlen_desc_t* desc, parse_work_item_t* out,
                                                 size_t capacity, size_t* n_items) {
  Problem p;
  std::string err;
  parse_status_t s = make_problem_varlen(desc, &p, &err);
  if (s != PARSE_OK) return fail(s, err);
  if (!n_items) return fail(PARSE_ERR_INVALID, "n_items is NULL");
  std::vector<WorkItem> items;
  build_schedule(p, &items);
  *n_items = items.size();
  if (out) std::memcpy(out, items.data(), sizeof(WorkItem) * std::min(capacity, items.size()));
  g_err.clear();
  return PARSE_OK;
}

namespace {
parse_status_t verify_varlen(const parse_varlen_desc_t* desc, const void* q, const void* k, const void* v, void* o,
                             float* lse, void* workspace, size_t workspace_bytes, void* stream_, int precision,
                             const float* descale) {
  Problem p;
  std::string err;
  parse_status_t s = make_problem_varlen(desc, &p, &err);
  if (s != PARSE_OK) return fail(s, err);
  // packed rows: TMA dims (d, head, row, 1); paged K/V: (d, head, row in page, page)
  VerifyIO io{};
  io.q = q; io.k = k; io.v = v; io.o = o; io.lse = lse;
  const int64_t T = desc->total_rows;
  io.q_geom = {T, 1, {T * desc->q_strides[0], desc->q_strides[0], desc->q_strides[1]}};
  if (desc->page_size) {
    io.page_log2 = 0;
    while ((1 << io.page_log2) < desc->page_size) ++io.page_log2;
    io.num_pages = desc->num_pages;
    io.block_table = desc->block_table;
    io.bt_stride = desc->block_table_stride;
    io.k_geom = {desc->page_size, desc->num_pages, {desc->k_strides[0], desc->k_strides[1], desc->k_strides[2]}};
    io.v_geom = {desc->page_size, desc->num_pages, {desc->v_strides[0], desc->v_strides[1], desc->v_strides[2]}};
  } else {
    const int64_t KT = desc->kv_row_offsets ? desc->kv_total_rows : T;
    io.k_geom = {KT, 1, {KT * desc->k_strides[0], desc->k_strides[0], desc->k_strides[1]}};
    io.v_geom = {KT, 1, {KT * desc->v_strides[0], desc->v_strides[0], desc->v_strides[1]}};
  }
  io.o_strides[0] = T * desc->o_strides[0];
  io.o_strides[1] = desc->o_strides[0];
  io.o_strides[2] = desc->o_strides[1];
  io.lse_sb = 0;
  io.lse_sh = T;
  if (descale)
    for (int i = 0; i < 3; ++i) io.descale[i] = descale[i];
  return launch_verify(p, precision, io, workspace, workspace_bytes, static_cast<cudaStream_t>(stream_));
}
}  // namespace

parse_status_t parse_verify_attn_varlen(const parse_varlen_desc_t* desc, const void* q, const void* k,
                                        const void* v, void* o, float* lse, void* workspace, size_t workspace_bytes,
                                        void* stream_) {
  if (desc && desc->precision == PARSE_PREC_FP8_E4M3)
    return fail(PARSE_ERR_INVALID, "PARSE_PREC_FP8_E4M3 inputs go through parse_verify_attn_varlen_fp8");
  return verify_varlen(desc, q, k, v, o, lse, workspace, workspace_bytes, stream_, desc ? desc->precision : 0,
                       nullptr);
}

parse_status_t parse_verify_attn_varlen_fp8(const parse_varlen_desc_t* desc, const void* q, const void* k,
                                            const void* v, float descale_q, float descale_k, float descale_v, void* o,
                                            float* lse, void* workspace, size_t workspace_bytes, void* stream_) {
  if (!desc) return fail(PARSE_ERR_INVALID, "desc is NULL");
  if (desc->precision != PARSE_PREC_FP8_E4M3)
    return fail(PARSE_ERR_INVALID, "desc->precision must be PARSE_PREC_FP8_E4M3");
  const int64_t* st[3] = {desc->q_strides, desc->k_strides, desc->v_strides};
  const int ns[3] = {2, 3, 3};
  for (int t = 0; t < 3; ++t)
    for (int i = 0; i < ns[t]; ++i)
      if (st[t][i] % 16) return fail(PARSE_ERR_INVALID, "FP8 q/k/v strides must be multiples of 16 elements");
  if (!(descale_q > 0.f) || !(descale_k > 0.f) || !(descale_v > 0.f) || !std::isfinite(descale_q) ||
      !std::isfinite(descale_k) || !std::isfinite(descale_v))
    return fail(PARSE_ERR_INVALID, "descale factors must be positive and finite");
  const float ds[3] = {descale_q, descale_k, descale_v};
  return verify_varlen(desc, q, k, v, o, lse, workspace, workspace_bytes, stream_, PARSE_PREC_FP8_E4M3, ds);
}

parse_status_t parse_select_prefix(const parse_select_desc_t* d, int32_t* accepted_len, int32_t* k_star,
                                   float* scores, parse_prefix_stats_t* stats, int32_t* device_status,
                                   void* stream_) {
  if (!d) return fail(PARSE_ERR_INVALID, "desc is NULL");
  if (d->batch < 1 || d->num_prefixes < 1 || d->num_prefixes > 65536)
    return fail(PARSE_ERR_INVALID, "need batch >= 1 and 1 <= num_prefixes <= 65536");
  if (!d->verdict_logits || !d->boundaries || !accepted_len || !k_star || !scores)
    return fail(PARSE_ERR_INVALID, "verdict_logits, boundaries, accepted_len, k_star, scores must be non-NULL");
  if (!(d->threshold >= 0.0 && d->threshold <= 1.0)) return fail(PARSE_ERR_INVALID, "threshold must be in [0, 1]");
  if (!(d->aux_threshold <= 1.0)) return fail(PARSE_ERR_INVALID, "aux_threshold must be <= 1");
  if (!(d->eta >= 0.0) || !std::isfinite(d->eta)) return fail(PARSE_ERR_INVALID, "eta must be finite and >= 0");
  if (d->rule != PARSE_RULE_LEADING_RUN && d->rule != PARSE_RULE_MAX_CORRECT)
    return fail(PARSE_ERR_INVALID, "unknown rule");
  if (d->logits_batch_stride < 0 || d->logits_prefix_stride < 0 || d->boundary_batch_stride < 0)
    return fail(PARSE_ERR_INVALID, "negative stride");
  DeviceInfo di;
  parse_status_t s;
  if ((s = check_device(&di)) != PARSE_OK) return s;
  SelectParams p{};
  p.logits = d->verdict_logits;
  p.bf16 = d->logits_bf16 ? 1 : 0;
  p.ls_b = d->logits_batch_stride; p.ls_k = d->logits_prefix_stride; p.ls_pair = d->logits_pair_stride;
  p.bnd = d->boundaries; p.bnd_s = d->boundary_batch_stride;
  p.B = d->batch; p.K = d->num_prefixes;
  p.theta = logit_threshold(d->threshold);
  p.use_aux = d->aux_threshold >= 0.0;
  p.theta_aux = p.use_aux ? logit_threshold(d->aux_threshold) : 0.0;
  p.eta = d->eta; p.rule = d->rule; p.tie = d->tie_is_correct ? 1 : 0;
  p.accepted = accepted_len; p.kstar = k_star; p.scores = scores; p.stats = stats; p.status = device_status;
  cudaError_t e = launch_select(p, static_cast<cudaStream_t>(stream_));
  if (e != cudaSuccess) return cuda_fail(e, "select launch");
  g_err.clear();
  return PARSE_OK;
}

// ---------------------------------------------------------------------------
// Fused select + all-gather over peer memory
// ---------------------------------------------------------------------------
namespace {
std::mutex g_peer_mu;
std::unordered_map<uintptr_t, uintptr_t> g_peer_bases;   // imported pointer -> mapped base

using PFN_getRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
PFN_getRange get_range_fn() {
  static PFN_getRange fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_getRange>(ptr);
  });
  return fn;
}
}  // namespace

parse_status_t parse_peer_buffer_bytes(int32_t batch, int32_t num_prefixes, int32_t world, size_t* bytes) {
  if (batch < 1 || num_prefixes < 1 || num_prefixes > 65536 || world < 1 || world > kPeerMaxWorld || !bytes)
    return fail(PARSE_ERR_INVALID, "need batch, num_prefixes >= 1 and 1 <= world <= 32");
  *bytes = size_t(kPeerHeader) + size_t(kPeerSets) * world * size_t(batch) * (2 + size_t(num_prefixes)) * 4;
  g_err.clear();
  return PARSE_OK;
}

parse_status_t parse_peer_export(const void* dev_ptr, parse_ipc_handle_t* handle, uint64_t* offset) {
  if (!dev_ptr || !handle || !offset) return fail(PARSE_ERR_INVALID, "NULL argument");
  auto rng = get_range_fn();
  if (!rng) return fail(PARSE_ERR_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (rng(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return fail(PARSE_ERR_INVALID, "dev_ptr is not device memory");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  static_assert(sizeof(cudaIpcMemHandle_t) <= sizeof(parse_ipc_handle_t), "handle size");
  std::memset(handle, 0, sizeof(*handle));
  std::memcpy(handle->reserved, &h, sizeof(h));
  *offset = uint64_t(reinterpret_cast<uintptr_t>(dev_ptr) - uintptr_t(base));
  g_err.clear();
  return PARSE_OK;
}

parse_status_t parse_peer_import(const parse_ipc_handle_t* handle, uint64_t offset, void** dev_ptr) {
  if (!handle || !dev_ptr) return fail(PARSE_ERR_INVALID, "NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle->reserved, sizeof(h));
  void* base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
  *dev_ptr = static_cast<uint8_t*>(base) + offset;
  std::lock_guard<std::mutex> lk(g_peer_mu);
  g_peer_bases[reinterpret_cast<uintptr_t>(*dev_ptr)] = reinterpret_cast<uintptr_t>(base);
  g_err.clear();
  return PARSE_OK;
}

parse_status_t parse_peer_close(void* dev_ptr) {
  uintptr_t base = 0;
  {
    std::lock_guard<std::mutex> lk(g_peer_mu);
    auto it = g_peer_bases.find(reinterpret_cast<uintptr_t>(dev_ptr));
    if (it == g_peer_bases.end()) return fail(PARSE_ERR_INVALID, "pointer was not returned by parse_peer_import");
    base = it->second;
    g_peer_bases.erase(it);
  }
  cudaError_t e = cudaIpcCloseMemHandle(reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcCloseMemHandle");
  g_err.clear();
  return PARSE_OK;
}

parse_status_t parse_select_prefix_allgather(const parse_select_desc_t* d, void* const* peer_buffers, int32_t rank,
                                             int32_t world, uint32_t epoch, parse_prefix_stats_t* stats,
                                             int32_t* device_status, void* stream_) {
  if (!d) return fail(PARSE_ERR_INVALID, "desc is NULL");
  if (world < 1 || world > kPeerMaxWorld || rank < 0 || rank >= world)
    return fail(PARSE_ERR_INVALID, "need 1 <= world <= 32 and 0 <= rank < world");
  if (!peer_buffers) return fail(PARSE_ERR_INVALID, "peer_buffers is NULL");
  if (epoch == 0) return fail(PARSE_ERR_INVALID, "epoch must be >= 1 (buffers start zeroed)");
  if (d->batch < 1 || d->num_prefixes < 1 || d->num_prefixes > 65536)
    return fail(PARSE_ERR_INVALID, "need batch >= 1 and 1 <= num_prefixes <= 65536");
  if (!d->verdict_logits || !d->boundaries)
    return fail(PARSE_ERR_INVALID, "verdict_logits, boundaries must be non-NULL");
  if (!(d->threshold >= 0.0 && d->threshold <= 1.0)) return fail(PARSE_ERR_INVALID, "threshold must be in [0, 1]");
  if (!(d->aux_threshold <= 1.0)) return fail(PARSE_ERR_INVALID, "aux_threshold must be <= 1");
  if (!(d->eta >= 0.0) || !std::isfinite(d->eta)) return fail(PARSE_ERR_INVALID, "eta must be finite and >= 0");
  if (d->rule != PARSE_RULE_LEADING_RUN && d->rule != PARSE_RULE_MAX_CORRECT)
    return fail(PARSE_ERR_INVALID, "unknown rule");
  if (d->logits_batch_stride < 0 || d->logits_prefix_stride < 0 || d->boundary_batch_stride < 0)
    return fail(PARSE_ERR_INVALID, "negative stride");
  DeviceInfo di;
  parse_status_t s;
  if ((s = check_device(&di)) != PARSE_OK) return s;
  SelectParams p{};
  p.logits = d->verdict_logits;
  p.bf16 = d->logits_bf16 ? 1 : 0;
  p.ls_b = d->logits_batch_stride; p.ls_k = d->logits_prefix_stride; p.ls_pair = d->logits_pair_stride;
  p.bnd = d->boundaries; p.bnd_s = d->boundary_batch_stride;
  p.B = d->batch; p.K = d->num_prefixes;
  p.theta = logit_threshold(d->threshold);
  p.use_aux = d->aux_threshold >= 0.0;
  p.theta_aux = p.use_aux ? logit_threshold(d->aux_threshold) : 0.0;
  p.eta = d->eta; p.rule = d->rule; p.tie = d->tie_is_correct ? 1 : 0;
  p.stats = stats; p.status = device_status;
  p.peers = reinterpret_cast<uint8_t* const*>(peer_buffers);
  p.rank = rank; p.world = world; p.epoch = epoch; p.set = int32_t(epoch % kPeerSets);
  p.slot_words = int64_t(d->batch) * (2 + d->num_prefixes);
  cudaError_t e = launch_select(p, static_cast<cudaStream_t>(stream_));
  if (e != cudaSuccess) return cuda_fail(e, "select launch");
  g_err.clear();
  return PARSE_OK;
}

parse_status_t parse_verdict_logits(const parse_verdict_head_desc_t* d, float* logits, void* stream_) {
  if (!d) return fail(PARSE_ERR_INVALID, "desc is NULL");
  if (d->batch < 1 || d->num_prefixes < 1 || d->hidden < 8 || d->hidden % 8)
    return fail(PARSE_ERR_INVALID, "need batch, num_prefixes >= 1 and hidden a positive multiple of 8");
  if (!d->hidden_states || !d->norm_weight || !d->verdict_rows || !logits)
    return fail(PARSE_ERR_INVALID, "hidden_states, norm_weight, verdict_rows, logits must be non-NULL");
  if (!(d->eps > 0.f)) return fail(PARSE_ERR_INVALID, "eps must be > 0");
  if (d->hs_batch_stride < 0 || d->hs_prefix_stride < 0 || (d->hs_batch_stride % 8) || (d->hs_prefix_stride % 8) ||
      !aligned16(d->hidden_states) || !aligned16(d->norm_weight) || !aligned16(d->verdict_rows))
    return fail(PARSE_ERR_INVALID, "hidden rows, gamma and W_U rows must be 16-byte aligned (strides % 8 == 0)");
  DeviceInfo di;
  parse_status_t s;
  if ((s = check_device(&di)) != PARSE_OK) return s;
  VerdictHeadParams p{};
  p.h = static_cast<const uint16_t*>(d->hidden_states);
  p.g = static_cast<const uint16_t*>(d->norm_weight);
  p.w = static_cast<const uint16_t*>(d->verdict_rows);
  p.hs_b = d->hs_batch_stride; p.hs_k = d->hs_prefix_stride;
  p.B = d->batch; p.K = d->num_prefixes; p.H = d->hidden; p.eps = d->eps;
  p.out = logits;
  cudaError_t e = launch_verdict_head(p, static_cast<cudaStream_t>(stream_));
  if (e != cudaSuccess) return cuda_fail(e, "verdict head launch");
  g_err.clear();
  return PARSE_OK;
}

parse_status_t parse_verdict_select(const parse_verdict_head_desc_t* hd, const parse_select_desc_t* sd, float* logits,
                                    uint32_t* counters, int32_t* accepted_len, int32_t* k_star, float* scores,
                                    parse_prefix_stats_t* stats, int32_t* device_status, void* stream_) {
  if (!hd || !sd) return fail(PARSE_ERR_INVALID, "desc is NULL");
  if (hd->batch < 1 || hd->num_prefixes < 1 || hd->hidden < 8 || hd->hidden % 8)
    return fail(PARSE_ERR_INVALID, "need batch, num_prefixes >= 1 and hidden a positive multiple of 8");
  if (sd->batch != hd->batch || sd->num_prefixes != hd->num_prefixes || hd->num_prefixes > 65536)
    return fail(PARSE_ERR_INVALID, "head and select descriptors must agree on batch and num_prefixes (<= 65536)");
  if (!hd->hidden_states || !hd->norm_weight || !hd->verdict_rows || !logits || !counters)
    return fail(PARSE_ERR_INVALID, "hidden_states, norm_weight, verdict_rows, logits, counters must be non-NULL");
  if (!sd->boundaries || !accepted_len || !k_star || !scores)
    return fail(PARSE_ERR_INVALID, "boundaries, accepted_len, k_star, scores must be non-NULL");
  if (!(hd->eps > 0.f)) return fail(PARSE_ERR_INVALID, "eps must be > 0");
  if (hd->hs_batch_stride < 0 || hd->hs_prefix_stride < 0 || (hd->hs_batch_stride % 8) || (hd->hs_prefix_stride % 8) ||
      !aligned16(hd->hidden_states) || !aligned16(hd->norm_weight) || !aligned16(hd->verdict_rows))
    return fail(PARSE_ERR_INVALID, "hidden rows, gamma and W_U rows must be 16-byte aligned (strides % 8 == 0)");
  if (!(sd->threshold >= 0.0 && sd->threshold <= 1.0)) return fail(PARSE_ERR_INVALID, "threshold must be in [0, 1]");
  if (!(sd->aux_threshold <= 1.0)) return fail(PARSE_ERR_INVALID, "aux_threshold must be <= 1");
  if (!(sd->eta >= 0.0) || !std::isfinite(sd->eta)) return fail(PARSE_ERR_INVALID, "eta must be finite and >= 0");
  if (sd->rule != PARSE_RULE_LEADING_RUN && sd->rule != PARSE_RULE_MAX_CORRECT)
    return fail(PARSE_ERR_INVALID, "unknown rule");
  if (sd->boundary_batch_stride < 0) return fail(PARSE_ERR_INVALID, "negative stride");
  DeviceInfo di;
  parse_status_t s;
  if ((s = check_device(&di)) != PARSE_OK) return s;
  VerdictHeadParams hp{};
  hp.h = static_cast<const uint16_t*>(hd->hidden_states);
  hp.g = static_cast<const uint16_t*>(hd->norm_weight);
  hp.w = static_cast<const uint16_t*>(hd->verdict_rows);
  hp.hs_b = hd->hs_batch_stride; hp.hs_k = hd->hs_prefix_stride;
  hp.B = hd->batch; hp.K = hd->num_prefixes; hp.H = hd->hidden; hp.eps = hd->eps;
  hp.out = logits;
  SelectParams sp{};
  sp.logits = logits; sp.bf16 = 0;
  sp.ls_b = 2 * int64_t(hd->num_prefixes); sp.ls_k = 2; sp.ls_pair = 1;   // the [B][K][2] buffer just written
  sp.bnd = sd->boundaries; sp.bnd_s = sd->boundary_batch_stride;
  sp.B = sd->batch; sp.K = sd->num_prefixes;
  sp.theta = logit_threshold(sd->threshold);
  sp.use_aux = sd->aux_threshold >= 0.0;
  sp.theta_aux = sp.use_aux ? logit_threshold(sd->aux_threshold) : 0.0;
  sp.eta = sd->eta; sp.rule = sd->rule; sp.tie = sd->tie_is_correct ? 1 : 0;
  sp.accepted = accepted_len; sp.kstar = k_star; sp.scores = scores; sp.stats = stats; sp.status = device_status;
  cudaError_t e = launch_verdict_select(hp, sp, counters, static_cast<cudaStream_t>(stream_));
  if (e != cudaSuccess) return cuda_fail(e, "verdict select launch");
  g_err.clear();
  return PARSE_OK;
}

parse_status_t parse_vocab_readout(const parse_vocab_readout_desc_t* d, float* pair_logits, float* lse,
                                   float* verdict_mass, void* stream_) {
  if (!d) return fail(PARSE_ERR_INVALID, "desc is NULL");
  const int per = d->logits_bf16 ? 8 : 4;
  if (d->batch < 1 || d->num_prefixes < 1 || d->vocab < per || d->vocab % per)
    return fail(PARSE_ERR_INVALID, "need batch, num_prefixes >= 1 and vocab a multiple of 8 (bf16) / 4 (fp32)");
  if (!d->vocab_logits || !pair_logits) return fail(PARSE_ERR_INVALID, "vocab_logits and pair_logits must be non-NULL");
  if (d->id_correct < 0 || d->id_correct >= d->vocab || d->id_incorrect < 0 || d->id_incorrect >= d->vocab)
    return fail(PARSE_ERR_INVALID, "token ids outside [0, vocab)");
  if (d->batch_stride < 0 || d->prefix_stride < 0 || (d->batch_stride % per) || (d->prefix_stride % per) ||
      !aligned16(d->vocab_logits))
    return fail(PARSE_ERR_INVALID, "vocab rows must be 16-byte aligned");
  DeviceInfo di;
  parse_status_t s;
  if ((s = check_device(&di)) != PARSE_OK) return s;
  VocabReadoutParams p{};
  p.z = d->vocab_logits; p.bf16 = d->logits_bf16 ? 1 : 0;
  p.s_b = d->batch_stride; p.s_k = d->prefix_stride;
  p.B = d->batch; p.K = d->num_prefixes; p.V = d->vocab; p.id_c = d->id_correct; p.id_i = d->id_incorrect;
  p.pair = pair_logits; p.lse = lse; p.mass = verdict_mass;
  cudaError_t e = launch_vocab_readout(p, static_cast<cudaStream_t>(stream_));
  if (e != cudaSuccess) return cuda_fail(e, "vocab readout launch");
  g_err.clear();
  return PARSE_OK;
}

}  // extern "C"
