// capi.cu — extern "C" entry points of libhetermoe_kernels.so (declared in include/hetermoe.h).
//
// Host-side responsibilities only: argument validation, TMA descriptor encoding
// (cuTensorMapEncodeTiled through the runtime's driver entry point; no -lcuda), grid sizing
// and launches on the caller's stream. No allocation, no synchronisation.
#include <atomic>
#include <vector>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>

#include "../../include/hetermoe.h"
#include "grouped_gemm.cuh"
#include "moe_kernels.cuh"

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

bool debug_sync() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("HM_DEBUG_SYNC");
    v = (s && atoi(s) != 0) ? 1 : 0;
  }
  return v == 1;
}

// HM_DEBUG_SYNC=1: synchronise the device after every launch so a fault is attributed to the
// kernel that caused it (debugging only; the default path never synchronises)
int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && debug_sync()) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return fail(static_cast<int>(e), "%s: %s", what, cudaGetErrorString(e));
  return 0;
}

// HM_PERMUTE_SPLIT (CTAs per 64-token permute chunk, 1..8), parsed once; 0 = not set. A value
// that is not an integer in range is reported on stderr once and ignored.
int permute_split_override() {
  static int v = -1;
  if (v < 0) {
    v = 0;
    if (const char* s = getenv("HM_PERMUTE_SPLIT")) {
      char* end = nullptr;
      const long n = strtol(s, &end, 10);
      if (end != s && *end == '\0' && n >= 1 && n <= 8) v = static_cast<int>(n);
      else fprintf(stderr, "hetermoe: ignoring HM_PERMUTE_SPLIT=%s (want 1..8)\n", s);
    }
  }
  return v;
}

// Opt a kernel into `smem` bytes of dynamic shared memory once per DEVICE (the attribute belongs
// to the device's context: a process that drives several GPUs must set it on each). `done` is the
// call site's bitmask of devices already set.
template <typename Kern>
int ensure_smem_attr(Kern kern, size_t smem, std::atomic<unsigned long long>& done, const char* what) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return 0;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return fail(static_cast<int>(e), "%s smem attr: %s", what, cudaGetErrorString(e));
  done.fetch_or(bit, std::memory_order_acq_rel);
  return 0;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// ---- TMA descriptor encoding -------------------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// bf16 tensor map with 128-byte swizzle. dims/strides innermost first; strides in bytes
// for dims 1..rank-1.
int make_map(CUtensorMap* m, const void* base, int rank, const uint64_t* dims,
             const uint64_t* strides_bytes, const uint32_t* box) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(HM_E_DRIVER, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base),
                  reinterpret_cast<const cuuint64_t*>(dims),
                  reinterpret_cast<const cuuint64_t*>(strides_bytes),
                  reinterpret_cast<const cuuint32_t*>(box), estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HM_E_SHAPE, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return 0;
}

int gemm_stats_enabled();
int gemm_ctas();

// Upper bound of a GEMM's tile count (the exact count depends on device-side expert sizes).
struct TileBound {
  bool group_k;
  long rows, M, N, E;
  long K = 0;  // reduction length (GROUP_M GEMMs)
  long tiles(long tile_m, long tile_n) const {
    const long ntl = (N + tile_n - 1) / tile_n;
    return group_k ? E * ((M + tile_m - 1) / tile_m) * ntl : (rows / tile_m + E) * ntl;
  }
};

template <bool GROUP_K, bool A_MN, bool B_MN, int EPI, int CTAS, int NSUB = 1, bool SHIFT = false>
int launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, const hm::GroupedGemmParams& p,
                const TileBound& tb, int max_ctas, cudaStream_t stream) {
  auto kern = hm::grouped_gemm_kernel<GROUP_K, A_MN, B_MN, EPI, CTAS, NSUB, SHIFT>;
  using Cfg = hm::TileCfg<CTAS, NSUB>;
  constexpr int smem = Cfg::kSmemBytes;
  const long ub_tiles = tb.tiles(Cfg::kTileM, Cfg::kTileN);
  static std::atomic<unsigned long long> attr_set{0};
  if (int rc = ensure_smem_attr(kern, smem, attr_set, "grouped_gemm")) return rc;
  // Default: one cluster per tile (upper bound `ub_tiles`), scheduled dynamically with cluster
  // launch control. A capacity cap (max_ctas > 0) instead runs a persistent grid of max_ctas
  // CTAs with static tile striding (the per-rank capacity-weight emulation).
  int grid;
  hm::GroupedGemmParams pp = p;
  pp.stats = gemm_stats_enabled();
  if (max_ctas > 0) {
    grid = max_ctas < num_sms() ? max_ctas : num_sms();
    grid = (grid / CTAS) * CTAS;
    if (grid < CTAS) grid = CTAS;
    pp.dynamic = 0;
  } else {
    long g = ub_tiles * CTAS;
    if (g < CTAS) g = CTAS;
    if (g > 0x7fffffffL) g = 0x7fffffffL / CTAS * CTAS;
    grid = static_cast<int>(g);
    pp.dynamic = 1;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(hm::kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = CTAS;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, pp);
  if (e != cudaSuccess) return fail(static_cast<int>(e), "grouped_gemm launch: %s", cudaGetErrorString(e));
  return check_launch("grouped_gemm");
}

int gemm_wide_mask();
bool gemm_wide_explicit();

// CTA count / tile width dispatch for one GEMM kind: 1 CTA (HM_GEMM_CTAS=1), a CTA pair with
// 256 x 256 tiles, or a CTA pair with 256 x 512 tiles (modes in the wide mask)
int gemm_group_m(int mode, long M);
int g_early_release = getenv("HM_GEMM_NO_EARLY_RELEASE") ? 0 : 1;

template <bool GROUP_K, bool A_MN, bool B_MN, int EPI, bool SHIFT = false>
int launch_kind(int mode, const CUtensorMap& ma, const CUtensorMap& mb, const hm::GroupedGemmParams& p0,
                const TileBound& tb, int max_ctas, cudaStream_t st) {
  hm::GroupedGemmParams p = p0;
  p.group_m = gemm_group_m(mode, tb.M);
  p.early_release = g_early_release;
  if (gemm_ctas() == 1) return launch_gemm<GROUP_K, A_MN, B_MN, EPI, 1, 1, SHIFT>(ma, mb, p, tb, max_ctas, st);
  bool wide = (gemm_wide_mask() >> mode) & 1;
  // the SwiGLU backward's drain-then-release epilogue holds the single wide accumulator for a
  // fixed few microseconds: worth it against a long K (C2, K = d = 4096: 1043 -> 1165 TFLOP/s),
  // not a short one (C3, K = 2048: 967 -> 764), unless HM_GEMM_WIDE forces the mask
  if (mode == HM_GEMM_BWD_DACT && !gemm_wide_explicit() && tb.K < 4096) wide = false;
  if (wide) return launch_gemm<GROUP_K, A_MN, B_MN, EPI, 2, 2, SHIFT>(ma, mb, p, tb, max_ctas, st);
  return launch_gemm<GROUP_K, A_MN, B_MN, EPI, 2, 1, SHIFT>(ma, mb, p, tb, max_ctas, st);
}

// raster group height per GEMM mode (HM_GEMM_GROUPM = one value for every mode; a negative value
// -g selects the transposed raster: groups of g n-tiles, n fastest). The per-mode defaults
// minimise DRAM traffic at equal time (C2 sweeps of 8/16/32/64 and -2/-4/-8/-16,
// profiles/r2_gemm_groupm.md): up+gate 32 (5.6 -> 3.6 GB read), SwiGLU backward 64, down and dX
// transposed in groups of 4 n-tiles (dX 8.2 -> 7.6 GB); the bf16 weight gradients 32 when the
// output has at most 32 row tiles (dW_d, M = d: 2.4 -> 1.6 GB), else transposed in groups of 8
// (dW_ug, M = 2f: 4.2 -> 2.7 GB); the fp32-accumulating multi-segment weight gradient of the ZP
// executor keeps 32 / 8.
int g_group_m[8] = {0, 0, 0, 0, 0, 0, 0, 0};
int gemm_group_m(int mode, long M = 0) {
  static const int kDefault[8] = {32, -4, 64, -4, 0, 0, 8, 8};  // by HM_GEMM_* mode; 0 = by M
  if (mode < 0 || mode >= 8) return hm::kGroupM;
  if (g_group_m[mode] == 0) {
    const char* s = getenv("HM_GEMM_GROUPM");
    const int v = s ? atoi(s) : 0;
    if (v != 0) g_group_m[mode] = v;
    else if (kDefault[mode] != 0) g_group_m[mode] = kDefault[mode];
    else if ((M + 255) / 256 <= 32) return 32;
    else return mode == HM_GEMM_WGRAD ? -8 : 8;
  }
  return g_group_m[mode];
}

int gemm_stats_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("HM_GEMM_STATS");
    v = (s && atoi(s) != 0) ? 1 : 0;
  }
  return v;
}

// GEMM modes (bit = HM_GEMM_* mode) that use the 256 x 512 "wide" pair tile; HM_GEMM_WIDE
// overrides the default (measured per mode on B200)
#ifndef HM_GEMM_WIDE_DEFAULT
#define HM_GEMM_WIDE_DEFAULT 0x3F  // every GEMM: up+gate, down, SwiGLU backward, dX, both wgrads
#endif
int g_wide_mask = -1;
bool g_wide_explicit = false;  // HM_GEMM_WIDE or hm_debug_set_gemm_wide chose the mask
int gemm_wide_mask() {
  if (g_wide_mask < 0) {
    const char* s = getenv("HM_GEMM_WIDE");
    g_wide_explicit = s != nullptr;
    g_wide_mask = s ? static_cast<int>(strtol(s, nullptr, 0)) : HM_GEMM_WIDE_DEFAULT;
  }
  return g_wide_mask;
}
bool gemm_wide_explicit() {
  gemm_wide_mask();
  return g_wide_explicit;
}

// CTA-pair (cta_group::2) tiles for the GROUP_M GEMMs unless HM_GEMM_CTAS=1
int gemm_ctas() {
  static int v = 0;
  if (v == 0) {
    const char* s = getenv("HM_GEMM_CTAS");
    v = (s && atoi(s) == 1) ? 1 : 2;
  }
  return v;
}

}  // namespace

// K1b: thread-per-token top-k for E % 4 == 0, E <= 64 (bit-identical to the warp-per-token
// kernel, which stays for E > 64 and for A/B runs via HM_TOPK_WARP).
static void launch_router_topk(int nchunk, cudaStream_t st, const float* logits, int T, int E, int k,
                               int32_t* idx, float* w, int32_t* chunk_base) {
  if (E % 4 == 0 && E <= 64 && !getenv("HM_TOPK_WARP")) {
    if (E <= 16) hm::router_topk_lane_kernel<16><<<nchunk, hm::kChunk, 0, st>>>(logits, T, E, k, idx, w, chunk_base);
    else if (E <= 32) hm::router_topk_lane_kernel<32><<<nchunk, hm::kChunk, 0, st>>>(logits, T, E, k, idx, w, chunk_base);
    else hm::router_topk_lane_kernel<64><<<nchunk, hm::kChunk, 0, st>>>(logits, T, E, k, idx, w, chunk_base);
  } else {
    hm::router_topk_kernel<<<nchunk, 512, 0, st>>>(logits, T, E, k, idx, w, chunk_base);
  }
}

extern "C" {

int hm_abi_version(void) { return HM_ABI_VERSION; }

// debugging aid (not part of the ABI): the per-expert wgrad TMA views as built on the device
// (first E*2 maps of `out`) next to the same views encoded on the host (next E*2 maps)
int hm_debug_expert_maps(const void* a, const void* b, const int32_t* seg_offsets, int E, int rows,
                         int M, int N, unsigned char* out) {
  CUtensorMap ma, mb;
  uint64_t dims_a[2] = {(uint64_t)M, (uint64_t)rows};
  uint64_t str_a[1] = {(uint64_t)M * 2};
  uint32_t box[2] = {64, 64};
  if (int rc = make_map(&ma, a, 2, dims_a, str_a, box)) return rc;
  uint64_t dims_b[2] = {(uint64_t)N, (uint64_t)rows};
  uint64_t str_b[1] = {(uint64_t)N * 2};
  if (int rc = make_map(&mb, b, 2, dims_b, str_b, box)) return rc;
  CUtensorMap* ws = nullptr;
  if (cudaMalloc(&ws, 2 * E * sizeof(CUtensorMap)) != cudaSuccess) return -1;
  hm::SegBases bases{};
  bases.a[0] = static_cast<const uint8_t*>(a);
  bases.b[0] = static_cast<const uint8_t*>(b);
  hm::build_expert_maps_kernel<<<(E + 127) / 128, 128>>>(ma, mb, seg_offsets, E, 1, bases,
                                                          static_cast<long>(M) * 2, static_cast<long>(N) * 2, ws);
  cudaDeviceSynchronize();
  cudaMemcpy(out, ws, 2 * E * sizeof(CUtensorMap), cudaMemcpyDeviceToHost);
  cudaFree(ws);
  int* seg = new int[E + 1];
  cudaMemcpy(seg, seg_offsets, (E + 1) * sizeof(int), cudaMemcpyDeviceToHost);
  CUtensorMap* host = reinterpret_cast<CUtensorMap*>(out) + 2 * E;
  for (int e = 0; e < E; ++e) {
    const int me = seg[e + 1] - seg[e];
    uint64_t da[2] = {(uint64_t)M, (uint64_t)(me > 0 ? me : 1)};
    uint64_t db[2] = {(uint64_t)N, (uint64_t)(me > 0 ? me : 1)};
    make_map(&host[2 * e], static_cast<const uint8_t*>(a) + (long)seg[e] * M * 2, 2, da, str_a, box);
    make_map(&host[2 * e + 1], static_cast<const uint8_t*>(b) + (long)seg[e] * N * 2, 2, db, str_b, box);
  }
  delete[] seg;
  return 0;
}

// debugging aid (not part of the ABI): the fused router's per-CTA phase stamps of the last
// launch (HM_ROUTER_TIMELINE builds only; zeros otherwise), 512 x 5 u64 into out
int hm_debug_router_timeline(unsigned long long* out) {
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpyFromSymbol(out, hm::g_router_tl, sizeof(hm::g_router_tl));
  return static_cast<int>(e);
}
// debugging aid (not part of the ABI): first out-of-range access recorded by an
// HM_BOUNDS_CHECK build of the grouped GEMM; reads and clears the record
int hm_debug_read(long long* out8) {
  cudaError_t e = cudaMemcpyFromSymbol(out8, hm::g_hm_dbg, 8 * sizeof(long long));
  if (e != cudaSuccess) return static_cast<int>(e);
  long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  return static_cast<int>(cudaMemcpyToSymbol(hm::g_hm_dbg, z, sizeof(z)));
}

// Read (and reset) the grouped-GEMM cycle accounting collected when HM_GEMM_STATS=1:
// out[0] MMA waiting on TMA, [1] MMA waiting on a free accumulator, [2] MMA role cycles,
// [3] producer waiting on free stages, [4] tiles, [5] CTAs. Synchronises the device.
int hm_gemm_stats(unsigned long long* out) {
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpyFromSymbol(out, hm::g_gemm_stats, 8 * sizeof(unsigned long long));
  unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(hm::g_gemm_stats, z, sizeof(z));
  if (e != cudaSuccess) return fail(static_cast<int>(e), "gemm_stats: %s", cudaGetErrorString(e));
  return 0;
}
// tuning aid (not part of the ABI): set the wide-tile GEMM mode mask (-1 = default / env) and
// return the previous one, so variants can be A/B-timed in one process
int hm_debug_set_gemm_wide(int mask) {
  const int old = gemm_wide_mask();
  g_wide_mask = mask;
  g_wide_explicit = mask >= 0;
  return old;
}
// tuning aid (not part of the ABI): raster group height of one GEMM mode (mode < 0: all modes;
// value == 0: back to the default; value < 0: the transposed raster, -value n-tiles per group);
// returns the previous value of `mode` (or of mode 0)
int hm_debug_set_gemm_groupm(int mode, int value) {
  const int old = gemm_group_m(mode < 0 ? 0 : mode, 0);
  for (int m = 0; m < 8; ++m)
    if (mode < 0 || m == mode) g_group_m[m] = value;
  return old;
}
// tuning aid (not part of the ABI): wide plain-store epilogue releases its accumulator early (1)
// or after every store (0); returns the previous setting
int hm_debug_set_gemm_early_release(int on) {
  const int old = g_early_release;
  g_early_release = on;
  return old;
}
const char* hm_last_error(void) { return g_last_error.c_str(); }
int hm_num_sms(void) { return num_sms(); }

// ---------------------------------------------------------------------------------------------
// Router plan for d (blocks of 256, up to 64): EGW experts per CTA group and BPW blocks per warp
// keep at most 64 fp32 router weights per thread in registers.
static bool router_shape(int d, int* egw, int* bpw) {
  if (d <= 0 || d % 256 != 0 || d / 256 > 64) return false;
  const int nj = d / 256;
  *bpw = (nj + 15) / 16;
  *egw = *bpw == 1 ? 8 : (*bpw == 2 ? 4 : 2);
  return true;
}

// HM_ROUTER_UNFUSED: logits kernel + separate top-k + scan even for one expert group (read on
// every call: tests switch it at run time to compare the two paths)
static bool router_unfused_forced() { return getenv("HM_ROUTER_UNFUSED") != nullptr; }

int hm_router_launches(int T, int d, int E) {
  int egw, bpw;
  if (T <= 0 || !router_shape(d, &egw, &bpw)) return 0;
  return (E <= egw && !router_unfused_forced()) ? 1 : 3;
}

size_t hm_router_chunk_elems(int T, int E) {
  // per-chunk counts / row bases, then the fused kernel's CTA completion counter
  const size_t nchunk = (static_cast<size_t>(T) + hm::kChunk - 1) / hm::kChunk;
  return nchunk * E + 1;
}

}  // extern "C"

template <int EGW, int NJ_T, int BPW, bool FUSE>
static int launch_router_fused(int groups, cudaStream_t st, const __nv_bfloat16* xb, const __nv_bfloat16* wb,
                               const float* bias, int T, int d, int E, float* logits, int k, int32_t* idx,
                               float* w, int32_t* chunk_base, int32_t* counts, int32_t* offsets) {
  auto kern = hm::router_fused_kernel<EGW, NJ_T, BPW, FUSE>;
  const size_t smem = hm::router_fused_smem_bytes(EGW);
  static std::atomic<unsigned long long> attr{0};
  if (int rc = ensure_smem_attr(kern, smem, attr, "router")) return rc;
  const int nj = d / 256;
  const int TG = nj <= 16 ? 4 * (16 / nj) : 4 / BPW;
  const int units = (T + TG - 1) / TG;
  int ranges = num_sms() / groups;  // one persistent CTA per SM over all (range, group) pairs
  if (ranges < 1) ranges = 1;
  if (ranges > units) ranges = units;
  kern<<<ranges * groups, hm::kRouterThreads, smem, st>>>(xb, wb, bias, T, d, E, ranges, logits, k, idx, w,
                                                          chunk_base, counts, offsets);
  return check_launch("router_fused");
}

// compile-time block counts for d = 256 * 2^m (every index a shift), run-time otherwise
template <bool FUSE>
static int launch_router_nj(int d, int groups, cudaStream_t st, const __nv_bfloat16* xb, const __nv_bfloat16* wb,
                            const float* bias, int T, int E, float* logits, int k, int32_t* idx, float* w,
                            int32_t* chunk_base, int32_t* counts, int32_t* offsets) {
#define HM_ROUTER_ARGS groups, st, xb, wb, bias, T, d, E, logits, k, idx, w, chunk_base, counts, offsets
  switch (d / 256) {
    case 1: return launch_router_fused<8, 1, 1, FUSE>(HM_ROUTER_ARGS);
    case 2: return launch_router_fused<8, 2, 1, FUSE>(HM_ROUTER_ARGS);
    case 4: return launch_router_fused<8, 4, 1, FUSE>(HM_ROUTER_ARGS);
    case 8: return launch_router_fused<8, 8, 1, FUSE>(HM_ROUTER_ARGS);
    case 16: return launch_router_fused<8, 16, 1, FUSE>(HM_ROUTER_ARGS);
    case 32: return launch_router_fused<4, 32, 2, FUSE>(HM_ROUTER_ARGS);
    case 64: return launch_router_fused<2, 64, 4, FUSE>(HM_ROUTER_ARGS);
    default: {
      const int bpw = (d / 256 + 15) / 16;
      if (bpw == 1) return launch_router_fused<8, 0, 1, FUSE>(HM_ROUTER_ARGS);
      if (bpw == 2) return launch_router_fused<4, 0, 2, FUSE>(HM_ROUTER_ARGS);
      if (bpw == 3) return launch_router_fused<2, 0, 3, FUSE>(HM_ROUTER_ARGS);
      return launch_router_fused<2, 0, 4, FUSE>(HM_ROUTER_ARGS);
    }
  }
#undef HM_ROUTER_ARGS
}

extern "C" {

int hm_router_topk(const void* x, const void* wg, const float* bias, int T, int d, int E, int k,
                   int32_t* idx, float* w, float* logits, int32_t* counts, int32_t* offsets,
                   int32_t* chunk_base, void* stream) {
  int egw = 0, bpw = 0;
  if (T < 0 || !router_shape(d, &egw, &bpw) || E < 1 || E > 256 || k < 1 || k > hm::kMaxTopK || k > E)
    return fail(HM_E_SHAPE, "router: unsupported shape T=%d d=%d E=%d k=%d (d %% 256 == 0, d <= 16384)", T, d, E, k);
  if (!aligned16(x)) return fail(HM_E_ALIGN, "router: x not 16-byte aligned");
  cudaStream_t st = S(stream);
  const int nchunk = (T + hm::kChunk - 1) / hm::kChunk;
  if (T == 0) {
    cudaMemsetAsync(counts, 0, sizeof(int32_t) * E, st);
    cudaMemsetAsync(offsets, 0, sizeof(int32_t) * (E + 1), st);
    return check_launch("router(empty)");
  }
  const __nv_bfloat16* xb = static_cast<const __nv_bfloat16*>(x);
  const __nv_bfloat16* wb = static_cast<const __nv_bfloat16*>(wg);
  const int groups = (E + egw - 1) / egw;
  if (groups == 1 && !router_unfused_forced()) {
    // logits, top-k, softmax, chunk histogram and scan in one kernel (the histogram accumulates
    // with atomics into the zeroed chunk table; the last CTA scans it)
    cudaMemsetAsync(chunk_base, 0, sizeof(int32_t) * hm_router_chunk_elems(T, E), st);
    return launch_router_nj<true>(d, 1, st, xb, wb, bias, T, E, logits, k, idx, w, chunk_base, counts, offsets);
  }
  if (int rc = launch_router_nj<false>(d, groups, st, xb, wb, bias, T, E, logits, 0, nullptr, nullptr, nullptr,
                                       nullptr, nullptr))
    return rc;
  launch_router_topk(nchunk, st, logits, T, E, k, idx, w, chunk_base);
  if (int rc2 = check_launch("router_topk")) return rc2;
  hm::router_scan_kernel<<<1, 1024, 0, st>>>(chunk_base, nchunk, E, counts, offsets);
  return check_launch("router_scan");
}

// ---------------------------------------------------------------------------------------------
int hm_dispatch_permute(const void* x, const int32_t* idx, const int32_t* chunk_base, int T, int d,
                        int E, int k, void* x_perm, int32_t* row_src, int32_t* row_of,
                        void* stream) {
  if (T < 0 || d <= 0 || d % 8 != 0 || E < 1 || E > 256 || k < 1 || k > hm::kMaxTopK)
    return fail(HM_E_SHAPE, "permute: unsupported shape T=%d d=%d E=%d k=%d", T, d, E, k);
  if (!aligned16(x) || !aligned16(x_perm)) return fail(HM_E_ALIGN, "permute: x/x_perm alignment");
  if (T == 0) return 0;
  cudaStream_t st = S(stream);
  const int nchunk = (T + hm::kChunk - 1) / hm::kChunk;
  auto xb = static_cast<const __nv_bfloat16*>(x);
  auto xp = static_cast<__nv_bfloat16*>(x_perm);
  // 4 CTAs per 64-token chunk: C2 0.077 -> 0.069 ms (89 % of HBM), C3 0.097 -> 0.094 ms
  // (tools/permute_bench.py); HM_PERMUTE_SPLIT overrides for A/B runs
  const int split = permute_split_override() ? permute_split_override() : 4;
#define HM_PERMUTE_CASE(V)                                                                      \
  case V:                                                                                       \
    hm::dispatch_permute_kernel<V><<<dim3(nchunk, split), 256, 0, st>>>(xb, idx, chunk_base, T, d, E, k, xp, \
                                                            row_src, row_of);                   \
    break;
  if (d % 256 == 0 && d / 256 <= 16) {
    switch (d / 256) {
      HM_PERMUTE_CASE(1)
      HM_PERMUTE_CASE(2)
      HM_PERMUTE_CASE(4)
      HM_PERMUTE_CASE(8)
      HM_PERMUTE_CASE(16)
      default:
        hm::dispatch_permute_generic_kernel<<<nchunk, 256, 0, st>>>(xb, idx, chunk_base, T, d, E,
                                                                    k, xp, row_src, row_of);
    }
  } else {
    hm::dispatch_permute_generic_kernel<<<nchunk, 256, 0, st>>>(xb, idx, chunk_base, T, d, E, k,
                                                                xp, row_src, row_of);
  }
#undef HM_PERMUTE_CASE
  return check_launch("dispatch_permute");
}

#define HM_K_SWITCH(k, CALL)                                \
  switch (k) {                                              \
    case 1: { constexpr int K = 1; CALL; } break;           \
    case 2: { constexpr int K = 2; CALL; } break;           \
    case 3: { constexpr int K = 3; CALL; } break;           \
    case 4: { constexpr int K = 4; CALL; } break;           \
    case 5: { constexpr int K = 5; CALL; } break;           \
    case 6: { constexpr int K = 6; CALL; } break;           \
    case 7: { constexpr int K = 7; CALL; } break;           \
    case 8: { constexpr int K = 8; CALL; } break;           \
    default: return fail(HM_E_SHAPE, "unsupported k=%d", k); \
  }

static int row_grid(int T) {
  const int warps = T;
  int blocks = (warps + 7) / 8;
  const int cap = num_sms() * 8;
  return blocks < cap ? (blocks > 0 ? blocks : 1) : cap;
}

int hm_unpermute_sum(const void* dx_perm, const int32_t* row_of, int T, int d, int k, void* dx,
                     void* stream) {
  if (T < 0 || d <= 0 || d % 8 != 0) return fail(HM_E_SHAPE, "unpermute: bad shape");
  if (!aligned16(dx_perm) || !aligned16(dx)) return fail(HM_E_ALIGN, "unpermute: alignment");
  if (T == 0) return 0;
  auto in = static_cast<const __nv_bfloat16*>(dx_perm);
  auto out = static_cast<__nv_bfloat16*>(dx);
  HM_K_SWITCH(k, (hm::unpermute_sum_kernel<K><<<row_grid(T), 256, 0, S(stream)>>>(in, row_of, T, d, out)));
  return check_launch("unpermute_sum");
}

int hm_combine(const void* y_perm, const int32_t* row_of, const float* w, int T, int d, int k,
               void* y, void* stream) {
  if (T < 0 || d <= 0 || d % 8 != 0) return fail(HM_E_SHAPE, "combine: bad shape");
  if (!aligned16(y_perm) || !aligned16(y)) return fail(HM_E_ALIGN, "combine: alignment");
  if (T == 0) return 0;
  auto in = static_cast<const __nv_bfloat16*>(y_perm);
  auto out = static_cast<__nv_bfloat16*>(y);
  HM_K_SWITCH(k, (hm::combine_kernel<K><<<row_grid(T), 256, 0, S(stream)>>>(in, row_of, w, T, d, out)));
  return check_launch("combine");
}

int hm_combine_bwd(const void* dy, const void* y_perm, const int32_t* row_of, const float* w,
                   int T, int d, int k, void* dy_perm, float* dw, void* stream) {
  if (T < 0 || d <= 0 || d % 8 != 0) return fail(HM_E_SHAPE, "combine_bwd: bad shape");
  if (!aligned16(dy) || !aligned16(y_perm) || !aligned16(dy_perm))
    return fail(HM_E_ALIGN, "combine_bwd: alignment");
  if (T == 0) return 0;
  auto g = static_cast<const __nv_bfloat16*>(dy);
  auto yp = static_cast<const __nv_bfloat16*>(y_perm);
  auto out = static_cast<__nv_bfloat16*>(dy_perm);
  HM_K_SWITCH(k, (hm::combine_bwd_kernel<K><<<row_grid(T), 256, 0, S(stream)>>>(g, yp, row_of, w, T, d, out, dw)));
  return check_launch("combine_bwd");
}

// the dlogit region of the router-backward workspace, padded to 64 floats so the dWg partials
// after it stay 16-byte aligned (router_wgrad_perm_kernel stores float4; T*k % 4 != 0 faulted)
// K splits of the router weight-gradient GEMM (E > 8): about two waves of 256-column tiles
static int router_wgrad_gemm_splits(int d) {
  const int ntiles = (d + 255) / 256;
  int s = (2 * num_sms() / 2) / ntiles;  // CTA pairs
  return s < 1 ? 1 : (s > 16 ? 16 : s);
}
static size_t router_bwd_dl_elems(int T, int k) {
  return (static_cast<size_t>(T) * k + 63) & ~static_cast<size_t>(63);
}

// token splits of the streamed router weight gradient: one CTA per SM over (column tile, split)
static int router_wgrad_stream_splits(int T, int d) {
  const int tiles = (d + hm::kWgCols - 1) / hm::kWgCols;
  int s = num_sms() / tiles;
  if (s < 1) s = 1;
  const int max_s = (T + hm::kWgTok - 1) / hm::kWgTok;
  return s < max_s ? s : (max_s > 0 ? max_s : 1);
}

size_t hm_router_bwd_part_elems(int T, int d, int E, int k) {
  // dlogit (token or permuted-row order, T*k padded), the per-token dlogit records (T*16: dense
  // row + slots, E <= 8), then the per-split dWg partials (at most one split per SM)
  int splits = hm::kWgSplit > hm::kWgTokSplit ? hm::kWgSplit : hm::kWgTokSplit;
  if (num_sms() > splits) splits = num_sms();
  return router_bwd_dl_elems(T, k) + static_cast<size_t>(T) * hm::kRbMeta + static_cast<size_t>(splits) * E * d;
}

int hm_router_bwd(const void* dx_perm, const int32_t* row_of, const int32_t* idx, const float* w,
                  const float* dw, const void* x, const void* x_perm, const int32_t* offsets, const void* wg_t,
                  int T, int d, int E, int k, void* dx, float* dlogit, void* dwg, float* part,
                  void* stream) {
  if (T < 0 || d <= 0 || d % 8 != 0 || E < 1 || E > 256) return fail(HM_E_SHAPE, "router_bwd: bad shape");
  if (!aligned16(dx_perm) || !aligned16(dx) || !aligned16(wg_t) || (dwg && !aligned16(x_perm)))
    return fail(HM_E_ALIGN, "router_bwd: alignment");
  cudaStream_t st = S(stream);
  if (T == 0) {
    if (dwg) cudaMemsetAsync(dwg, 0, static_cast<size_t>(d) * E * 2, st);
    return check_launch("router_bwd(empty)");
  }
  if (dwg && (!part || !offsets || !x_perm)) return fail(HM_E_ARG, "router_bwd: dwg needs x_perm, offsets and part");
  auto dp = static_cast<const __nv_bfloat16*>(dx_perm);
  auto gt = static_cast<const __nv_bfloat16*>(wg_t);
  auto out = static_cast<__nv_bfloat16*>(dx);
  // dWg: for E <= 8 and the token rows x given, streamed token-major through shared memory from
  // the dense dlogit rows (each token row read once, contiguously); else token-major from the
  // first routed copies (k <= 3), else per expert over the permuted rows (each copy read once)
  const bool perm_forced = getenv("HM_ROUTER_WGRAD_PERM") != nullptr;
  // HM_ROUTER_BWD_FUSED=1 (E <= 8, k <= 3, with the token rows): the whole backward in one
  // streamed pass (dlogit records, then dx and the dWg partials per 1024-column tile, then the
  // split reduction). 0.116 vs 0.122 ms alone, but 0.170 vs 0.162 ms inside the C2 step
  // (tools/router_instep.py: both paths then pay the previous GEMM's L2 write-backs), so the
  // two-pass path below stays the default.
  if (dwg && E <= 8 && k <= 3 && x && d % hm::kRbCols == 0 && aligned16(x) && !perm_forced &&
      getenv("HM_ROUTER_BWD_FUSED") && !getenv("HM_ROUTER_WGRAD_TOK") && !getenv("HM_UNPERMUTE_V1") &&
      !getenv("HM_UNPERMUTE_V2") && !getenv("HM_UNPERMUTE_V3")) {
    float* meta = part + router_bwd_dl_elems(T, k);  // T * 16 floats (the T*8 region + partial space)
    float* partials = meta + static_cast<size_t>(T) * hm::kRbMeta;
    const int tiles = d / hm::kRbCols;
    int S = num_sms() / tiles;
    if (S < 1) S = 1;
    if (S > (T + hm::kRbTok - 1) / hm::kRbTok) S = (T + hm::kRbTok - 1) / hm::kRbTok;
    HM_K_SWITCH(k, (hm::router_dlogit_kernel<K><<<(T + 255) / 256, 256, 0, st>>>(idx, w, dw, T, meta, dlogit)));
    if (int rc = check_launch("router_dlogit")) return rc;
    auto launch = [&](auto kern, size_t smem) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kern<<<dim3(tiles, S), 17 * 32, smem, st>>>(dp, row_of, meta, static_cast<const __nv_bfloat16*>(x), gt, T, d, E,
                                                   out, partials);
    };
    if (k == 1) launch(hm::router_bwd_fused_kernel<1>, hm::RbCfg<1>::kSmem);
    else if (k == 2) launch(hm::router_bwd_fused_kernel<2>, hm::RbCfg<2>::kSmem);
    else launch(hm::router_bwd_fused_kernel<3>, hm::RbCfg<3>::kSmem);
    if (int rc = check_launch("router_bwd_fused")) return rc;
    const long n = static_cast<long>(d) * E;
    hm::router_wgrad_reduce_kernel<<<(n + 255) / 256, 256, 0, st>>>(partials, S, d, E, static_cast<__nv_bfloat16*>(dwg));
    return check_launch("router_wgrad_reduce");
  }
  const bool streamed = dwg && E <= 8 && x && d % hm::kWgCols == 0 && aligned16(x) && !perm_forced &&
                        !getenv("HM_ROUTER_WGRAD_TOK");
  // E > 8 with the token rows: dWg^T = dl^T . x as a K-split tensor-core GEMM (K3 WGRAD_ACC into
  // fp32 split partials over S token ranges, then the split reduction), from dense bf16 dlogit rows
  const size_t dl_el = router_bwd_dl_elems(T, k);
  const int wg_splits = router_wgrad_gemm_splits(d);
  const size_t dense_el = ((static_cast<size_t>(T) * E / 2) + 63) & ~static_cast<size_t>(63);
  const size_t gemm_need = dl_el + dense_el + 64 + 2 * 32 * wg_splits + 32 + static_cast<size_t>(wg_splits) * E * d;
  const bool gemm_wg = dwg && E > 8 && E % 8 == 0 && x && aligned16(x) && !perm_forced &&
                       !getenv("HM_ROUTER_WGRAD_TOK") && gemm_need <= hm_router_bwd_part_elems(T, d, E, k);
  const bool tok = dwg && !streamed && E <= 8 && k <= 3 && d % 64 == 0 && !perm_forced;
  float* dl_perm = (dwg && !tok && !streamed && !gemm_wg) ? part : nullptr;
  float* dl_tok = dlogit ? dlogit : ((tok || gemm_wg) ? part : nullptr);
  float* coef8 = streamed ? part + router_bwd_dl_elems(T, k) : nullptr;
  // k >= 4: metadata broadcast by shuffles, no row prefetch (C3, k = 6: 0.099 vs 0.121 ms);
  // k <= 3: the v1 kernel (C2, k = 2: 0.080 vs 0.088 ms). Both produce bit-identical dx / dlogit
  // (tools/router_bench.py). HM_UNPERMUTE_V1 / HM_UNPERMUTE_V2 force a variant for A/B runs.
  const bool v1 = getenv("HM_UNPERMUTE_V1") || (k <= 3 && !getenv("HM_UNPERMUTE_V3"));
  if (getenv("HM_UNPERMUTE_V2")) {
    HM_K_SWITCH(k, (hm::unpermute_router_bwd2_kernel<K, true><<<row_grid(T), 256, 0, st>>>(dp, row_of, idx, w, dw, gt, T, d, out, dl_tok, dl_perm, coef8)));
  } else if (v1) {
    HM_K_SWITCH(k, (hm::unpermute_router_bwd_kernel<K><<<row_grid(T), 256, 0, st>>>(dp, row_of, idx, w, dw, gt, T, d, out, dl_tok, dl_perm, coef8)));
  } else {
    HM_K_SWITCH(k, (hm::unpermute_router_bwd2_kernel<K, false><<<row_grid(T), 256, 0, st>>>(dp, row_of, idx, w, dw, gt, T, d, out, dl_tok, dl_perm, coef8)));
  }
  if (int rc = check_launch("unpermute_router_bwd")) return rc;
  if (streamed) {
    float* partials = coef8 + static_cast<size_t>(T) * 8;
    const int S = router_wgrad_stream_splits(T, d);
    const size_t smem = hm::router_wgrad_stream_smem_bytes();
    static std::atomic<unsigned long long> attr{0};
    if (int rc = ensure_smem_attr(hm::router_wgrad_stream_kernel, smem, attr, "router_wgrad_stream")) return rc;
    hm::router_wgrad_stream_kernel<<<dim3(d / hm::kWgCols, S), hm::kWgThreads, smem, st>>>(
        static_cast<const __nv_bfloat16*>(x), coef8, T, d, E, partials);
    if (int rc = check_launch("router_wgrad_stream")) return rc;
    const long n = static_cast<long>(d) * E;
    hm::router_wgrad_reduce_kernel<<<(n + 255) / 256, 256, 0, st>>>(partials, S, d, E, static_cast<__nv_bfloat16*>(dwg));
    return check_launch("router_wgrad_reduce");
  }
  if (gemm_wg) {
    const int S = wg_splits;
    auto* dense = reinterpret_cast<__nv_bfloat16*>(part + dl_el);
    auto* seg = reinterpret_cast<int32_t*>(part + dl_el + dense_el);
    // 128-byte aligned workspace for the per-split TMA views, then the fp32 split partials
    uintptr_t wsa = reinterpret_cast<uintptr_t>(part + dl_el + dense_el + 64);
    wsa = (wsa + 127) & ~static_cast<uintptr_t>(127);
    void* ws = reinterpret_cast<void*>(wsa);
    float* partials = reinterpret_cast<float*>(wsa + 2 * 128 * S + 128);
    const long nchunk = static_cast<long>(T) * (E / 8);
    HM_K_SWITCH(k, (hm::dense_dlogit_kernel<K><<<static_cast<int>((nchunk + 255) / 256 > 0 ? (nchunk + 255) / 256 : 1),
                                               256, 0, st>>>(idx, dl_tok, T, E, S, dense, seg)));
    if (int rc = check_launch("dense_dlogit")) return rc;
    cudaMemsetAsync(partials, 0, sizeof(float) * static_cast<size_t>(S) * E * d, st);
    if (int rc = hm_grouped_gemm(HM_GEMM_WGRAD_ACC, dense, x, seg, S, T, E, d, 0, partials, d, nullptr, 0,
                                 nullptr, 0, ws, 0, stream))
      return rc;
    const long n = static_cast<long>(d) * E;
    hm::router_wgrad_reduce_kernel<<<(n + 255) / 256, 256, 0, st>>>(partials, S, d, E, static_cast<__nv_bfloat16*>(dwg));
    return check_launch("router_wgrad_reduce");
  }
  if (tok) {
    float* partials = part + router_bwd_dl_elems(T, k);
    auto xp = static_cast<const __nv_bfloat16*>(x_perm);
    const dim3 grid(d / 64, hm::kWgTokSplit);
    if (k == 1) hm::router_wgrad_tok_kernel<1><<<grid, 256, 0, st>>>(xp, row_of, idx, dl_tok, T, d, E, partials);
    else if (k == 2) hm::router_wgrad_tok_kernel<2><<<grid, 256, 0, st>>>(xp, row_of, idx, dl_tok, T, d, E, partials);
    else hm::router_wgrad_tok_kernel<3><<<grid, 256, 0, st>>>(xp, row_of, idx, dl_tok, T, d, E, partials);
    if (int rc = check_launch("router_wgrad_tok")) return rc;
    const long n = static_cast<long>(d) * E;
    hm::router_wgrad_reduce_kernel<<<(n + 255) / 256, 256, 0, st>>>(
        partials, hm::kWgTokSplit, d, E, static_cast<__nv_bfloat16*>(dwg));
    return check_launch("router_wgrad_reduce");
  }
  if (dwg) {
    float* partials = part + router_bwd_dl_elems(T, k);
    dim3 grid(E * hm::kWgSplit, (d + 2047) / 2048);
    hm::router_wgrad_perm_kernel<<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x_perm),
                                                       dl_perm, offsets, d, E, partials);
    if (int rc = check_launch("router_wgrad_perm")) return rc;
    const long n = static_cast<long>(d) * E;
    hm::router_wgrad_reduce_kernel<<<(n + 255) / 256, 256, 0, st>>>(
        partials, hm::kWgSplit, d, E, static_cast<__nv_bfloat16*>(dwg));
    return check_launch("router_wgrad_reduce");
  }
  return 0;
}

int hm_dispatch_permute_p2p(const void* x, const int32_t* idx, const int32_t* chunk_base,
                            const int32_t* offsets, int T, int d, int E, int k, void* x_perm,
                            int32_t* row_src, int32_t* row_of, const unsigned long long* dest_base,
                            const int32_t* dest_start, void* stream) {
  if (T < 0 || d <= 0 || d % 8 != 0 || E < 1 || E > 256 || k < 1 || k > hm::kMaxTopK)
    return fail(HM_E_SHAPE, "permute_p2p: unsupported shape T=%d d=%d E=%d k=%d", T, d, E, k);
  if (!aligned16(x) || (x_perm && !aligned16(x_perm))) return fail(HM_E_ALIGN, "permute_p2p: alignment");
  if (T == 0) return 0;
  cudaStream_t st = S(stream);
  const int nchunk = (T + hm::kChunk - 1) / hm::kChunk;
  auto xb = static_cast<const __nv_bfloat16*>(x);
  auto xp = static_cast<__nv_bfloat16*>(x_perm);
  // default 1 CTA per chunk here: with 4 the ZP stack measured 0.689M / 1.432M tok/s at 2 / 4
  // GPUs against 0.695M / 1.447M with 1 (within box noise, not a gain); HM_PERMUTE_SPLIT overrides
  const int split = permute_split_override() ? permute_split_override() : 1;
#define HM_P2P_CASE(V)                                                                        \
  case V:                                                                                     \
    hm::dispatch_permute_p2p_kernel<V><<<dim3(nchunk, split), 256, 0, st>>>(xb, idx, chunk_base, offsets, T, d, \
                                                                E, k, xp, row_src, row_of,    \
                                                                dest_base, dest_start);       \
    break;
  switch (d % 256 == 0 ? d / 256 : 0) {
    HM_P2P_CASE(1)
    HM_P2P_CASE(2)
    HM_P2P_CASE(4)
    HM_P2P_CASE(8)
    HM_P2P_CASE(16)
    default:  // any other d % 8 == 0
      HM_P2P_CASE(0)
  }
#undef HM_P2P_CASE
  return check_launch("dispatch_permute_p2p");
}

int hm_combine_bwd_p2p(const void* dy, const void* y_perm, const int32_t* row_of, const int32_t* idx,
                       const float* w, const int32_t* offsets, int T, int d, int k,
                       const unsigned long long* dest_base, const int32_t* dest_start, float* dw,
                       void* stream) {
  if (T < 0 || d <= 0 || d % 8 != 0) return fail(HM_E_SHAPE, "combine_bwd_p2p: bad shape");
  if (!aligned16(dy) || !aligned16(y_perm)) return fail(HM_E_ALIGN, "combine_bwd_p2p: alignment");
  if (T == 0) return 0;
  auto g = static_cast<const __nv_bfloat16*>(dy);
  auto yp = static_cast<const __nv_bfloat16*>(y_perm);
  HM_K_SWITCH(k, (hm::combine_bwd_p2p_kernel<K><<<row_grid(T), 256, 0, S(stream)>>>(g, yp, row_of, idx, w, offsets, T, d, dest_base, dest_start, dw)));
  return check_launch("combine_bwd_p2p");
}

int hm_zp_layout(const int32_t* counts_all, int M, int E, const int32_t* owners, int me, int n_own,
                 int cap, const unsigned long long* y_base, long long dx_delta, int row_bytes,
                 int32_t* dest_start, int32_t* seg, unsigned long long* out_rows_y,
                 unsigned long long* out_rows_dx, int32_t* shifts, int32_t* top, int pool_base,
                 int pool_rows, int32_t* err, void* stream) {
  if (M < 1 || M > hm::kZpMaxSenders || E < 1 || E > 256 || me < 0 || me >= hm::kZpMaxPeersLayout || cap < 0 ||
      n_own < 0 || n_own > E || pool_base < 0 || pool_rows < 0)
    return fail(HM_E_SHAPE, "zp_layout: M=%d E=%d me=%d n_own=%d cap=%d", M, E, me, n_own, cap);
  if (!counts_all || !owners || (me < M && !dest_start) || !err ||
      (n_own > 0 && (!seg || !out_rows_y || !out_rows_dx || !shifts || !top || !y_base)))
    return fail(HM_E_ARG, "zp_layout: null argument");
  const int grid = cap > 0 ? (cap + hm::kZpLayoutRowsPerCta - 1) / hm::kZpLayoutRowsPerCta : 1;
  hm::zp_layout_kernel<<<grid, hm::kZpLayoutThreads, 0, S(stream)>>>(
      counts_all, M, E, owners, me, n_own, cap, y_base, dx_delta, row_bytes, dest_start, seg, out_rows_y,
      out_rows_dx, shifts, top, pool_base, pool_rows, err);
  return check_launch("zp_layout");
}

int hm_signal_peers(const unsigned long long* flag_ptrs, int n, void* stream) {
  if (n < 0 || n > hm::kMaxPeers) return fail(HM_E_ARG, "signal_peers: n=%d", n);
  if (n == 0) return 0;
  hm::PeerFlags f{};
  for (int i = 0; i < n; ++i) f.ptr[i] = flag_ptrs[i];
  hm::signal_add_kernel<<<1, 32, 0, S(stream)>>>(f, n);
  return check_launch("signal_peers");
}

int hm_wait_flags(const unsigned int* flags, int stride, const unsigned int* targets, int n,
                  void* stream) {
  if (n < 0 || n > hm::kMaxPeers) return fail(HM_E_ARG, "wait_flags: n=%d", n);
  if (n == 0) return 0;
  hm::FlagTargets t{};
  for (int i = 0; i < n; ++i) t.v[i] = targets[i];
  hm::wait_geq_kernel<<<1, 32, 0, S(stream)>>>(flags, stride, t, n);
  return check_launch("wait_flags");
}

int hm_transpose_bf16(const void* in, int R, int C, void* out, void* stream) {
  if (R <= 0 || C <= 0) return fail(HM_E_SHAPE, "transpose: bad shape");
  dim3 grid((C + 31) / 32, (R + 31) / 32);
  hm::transpose_bf16_kernel<<<grid, dim3(32, 8), 0, S(stream)>>>(
      static_cast<const __nv_bfloat16*>(in), R, C, static_cast<__nv_bfloat16*>(out));
  return check_launch("transpose_bf16");
}

// ---------------------------------------------------------------------------------------------
size_t hm_grouped_gemm_workspace_bytes(int mode, int E) {
  return (mode == HM_GEMM_WGRAD || mode == HM_GEMM_WGRAD_ACC) ? static_cast<size_t>(2 * E) * sizeof(CUtensorMap) : 0;
}

int hm_grouped_gemm_rows(int mode, const void* a, const void* b, const int32_t* seg_offsets,
                         int E, int rows, int M, int N, int K, void* out, int ldo, void* out2,
                         int ldo2, const void* aux, int ld_aux, void* workspace,
                         const unsigned long long* out_rows, int max_ctas, void* stream);

int hm_grouped_gemm(int mode, const void* a, const void* b, const int32_t* seg_offsets, int E,
                    int rows, int M, int N, int K, void* out, int ldo, void* out2, int ldo2,
                    const void* aux, int ld_aux, void* workspace, int max_ctas, void* stream) {
  return hm_grouped_gemm_rows(mode, a, b, seg_offsets, E, rows, M, N, K, out, ldo, out2, ldo2, aux,
                              ld_aux, workspace, nullptr, max_ctas, stream);
}

int hm_grouped_gemm_rows(int mode, const void* a, const void* b, const int32_t* seg_offsets,
                         int E, int rows, int M, int N, int K, void* out, int ldo, void* out2,
                         int ldo2, const void* aux, int ld_aux, void* workspace,
                         const unsigned long long* out_rows, int max_ctas, void* stream) {
  return hm_grouped_gemm_shifted(mode, a, b, seg_offsets, E, rows, 0, M, N, K, out, ldo, out2, ldo2, aux,
                                 ld_aux, workspace, out_rows, nullptr, max_ctas, stream);
}

int hm_grouped_gemm_shifted(int mode, const void* a, const void* b, const int32_t* seg_offsets,
                            int E, int rows, int a_rows, int M, int N, int K, void* out, int ldo,
                            void* out2, int ldo2, const void* aux, int ld_aux, void* workspace,
                            const unsigned long long* out_rows, const int32_t* row_shift,
                            int max_ctas, void* stream) {
  if (mode < HM_GEMM_FWD_UPGATE || mode > HM_GEMM_WGRAD_ACC) return fail(HM_E_ARG, "gemm: unknown mode %d", mode);
  if (E < 1 || E > hm::kMaxExperts) return fail(HM_E_SHAPE, "gemm: E=%d out of range", E);
  if (rows < 0 || N <= 0 || N % 8 != 0) return fail(HM_E_SHAPE, "gemm: bad rows/N");
  if (!aligned16(a) || !aligned16(b) || (!out_rows && !aligned16(out))) return fail(HM_E_ALIGN, "gemm: alignment");
  if (out_rows && mode != HM_GEMM_FWD_DOWN && mode != HM_GEMM_BWD_DX)
    return fail(HM_E_ARG, "gemm: per-row destinations only for the plain-store GEMMs");
  if (ldo % 8 != 0) return fail(HM_E_ALIGN, "gemm: ldo must be a multiple of 8");
  cudaStream_t st = S(stream);
  const bool wgrad = (mode == HM_GEMM_WGRAD || mode == HM_GEMM_WGRAD_ACC);
  if (wgrad && (workspace == nullptr || (reinterpret_cast<uintptr_t>(workspace) & 127u)))
    return fail(HM_E_ARG, "gemm: wgrad needs a 128-byte aligned workspace of hm_grouped_gemm_workspace_bytes()");
  if (!wgrad && (K <= 0 || K % 8 != 0)) return fail(HM_E_SHAPE, "gemm: K must be a positive multiple of 8");
  if (wgrad && (M <= 0 || M % 8 != 0)) return fail(HM_E_SHAPE, "gemm: M must be a positive multiple of 8");
  if (rows == 0 && !wgrad) return 0;
  if (row_shift && (wgrad || (reinterpret_cast<uintptr_t>(row_shift) & 7u)))
    return fail(HM_E_ARG, "gemm: row_shift is an 8-byte aligned int[2], GROUP_M modes only");
  if (a_rows < rows) a_rows = rows;

  hm::GroupedGemmParams p{};
  p.row_shift = row_shift;
  p.R = 1;
  p.seg_offsets = seg_offsets;
  p.E = E;
  p.M = M;
  p.N = N;
  p.K = K;
  p.out = static_cast<__nv_bfloat16*>(out);
  p.out_f32 = static_cast<float*>(out);
  p.out_rows = out_rows;
  p.ldo = ldo;
  p.out2 = static_cast<__nv_bfloat16*>(out2);
  p.ldo2 = ldo2;
  p.aux = static_cast<const __nv_bfloat16*>(aux);
  p.ld_aux = ld_aux;

  CUtensorMap ma, mb;
  const int rows_m = rows > 0 ? rows : 1;
  const int ctas = gemm_ctas();
  if (!wgrad) {
    {
      uint64_t dims[2] = {(uint64_t)K, (uint64_t)(a_rows > 0 ? a_rows : rows_m)};
      uint64_t str[1] = {(uint64_t)K * 2};
      uint32_t box[2] = {64, 128};
      if (int rc = make_map(&ma, a, 2, dims, str, box)) return rc;
    }
    const bool b_mn = (mode == HM_GEMM_BWD_DACT || mode == HM_GEMM_BWD_DX);
    if (!b_mn) {
      uint64_t dims[3] = {(uint64_t)K, (uint64_t)N, (uint64_t)E};
      uint64_t str[2] = {(uint64_t)K * 2, (uint64_t)N * K * 2};
      uint32_t box[3] = {64, (uint32_t)(256 / ctas), 1};
      if (int rc = make_map(&mb, b, 3, dims, str, box)) return rc;
    } else {
      uint64_t dims[3] = {(uint64_t)N, (uint64_t)K, (uint64_t)E};
      uint64_t str[2] = {(uint64_t)N * 2, (uint64_t)K * N * 2};
      uint32_t box[3] = {64, 64, 1};
      if (int rc = make_map(&mb, b, 3, dims, str, box)) return rc;
    }
  } else {
    uint64_t dims_a[2] = {(uint64_t)M, (uint64_t)rows_m};
    uint64_t str_a[1] = {(uint64_t)M * 2};
    uint32_t box[2] = {64, 64};
    if (int rc = make_map(&ma, a, 2, dims_a, str_a, box)) return rc;
    uint64_t dims_b[2] = {(uint64_t)N, (uint64_t)rows_m};
    uint64_t str_b[1] = {(uint64_t)N * 2};
    if (int rc = make_map(&mb, b, 2, dims_b, str_b, box)) return rc;
    // per-expert views (device side, no host sync on the expert sizes)
    CUtensorMap* maps = static_cast<CUtensorMap*>(workspace);
    hm::SegBases bases{};
    bases.a[0] = static_cast<const uint8_t*>(a);
    bases.b[0] = static_cast<const uint8_t*>(b);
    hm::build_expert_maps_kernel<<<(E + 127) / 128, 128, 0, st>>>(
        ma, mb, seg_offsets, E, 1, bases, static_cast<long>(M) * 2, static_cast<long>(N) * 2, maps);
    if (int rc = check_launch("build_expert_maps")) return rc;
    p.expert_maps = maps;
  }

  p.out_elems = wgrad ? static_cast<long>(E) * M * ldo : static_cast<long>(rows) * ldo;
  const TileBound tb{wgrad, rows, M, N, E, K};
  switch (mode) {
    // pool-placed operands (row_shift) run their own instantiation, so the plain GEMMs compile
    // exactly as without the feature
    case HM_GEMM_FWD_UPGATE:
      if (N % 256 != 0 || !out2) return fail(HM_E_SHAPE, "upgate: N=2f must be a multiple of 256 and h given");
      return row_shift ? launch_kind<false, false, false, hm::EPI_SWIGLU_FWD, true>(mode, ma, mb, p, tb, max_ctas, st)
                       : launch_kind<false, false, false, hm::EPI_SWIGLU_FWD>(mode, ma, mb, p, tb, max_ctas, st);
    case HM_GEMM_FWD_DOWN:
      return row_shift ? launch_kind<false, false, false, hm::EPI_STORE, true>(mode, ma, mb, p, tb, max_ctas, st)
                       : launch_kind<false, false, false, hm::EPI_STORE>(mode, ma, mb, p, tb, max_ctas, st);
    case HM_GEMM_BWD_DACT:
      if (N % 128 != 0 || !aux) return fail(HM_E_SHAPE, "dact: N=f must be a multiple of 128 and h given");
      return row_shift ? launch_kind<false, false, true, hm::EPI_SWIGLU_BWD, true>(mode, ma, mb, p, tb, max_ctas, st)
                       : launch_kind<false, false, true, hm::EPI_SWIGLU_BWD>(mode, ma, mb, p, tb, max_ctas, st);
    case HM_GEMM_BWD_DX:
      return row_shift ? launch_kind<false, false, true, hm::EPI_STORE, true>(mode, ma, mb, p, tb, max_ctas, st)
                       : launch_kind<false, false, true, hm::EPI_STORE>(mode, ma, mb, p, tb, max_ctas, st);
    case HM_GEMM_WGRAD:
      return launch_kind<true, true, true, hm::EPI_STORE>(mode, ma, mb, p, tb, max_ctas, st);
    case HM_GEMM_WGRAD_ACC:
      return launch_kind<true, true, true, hm::EPI_ACC_F32>(mode, ma, mb, p, tb, max_ctas, st);
    default:
      return fail(HM_E_ARG, "gemm: unknown mode %d", mode);
  }
}

size_t hm_grouped_wgrad_multi_workspace_bytes(int E, int R) {
  return static_cast<size_t>(2 * E) * R * sizeof(CUtensorMap);
}

int hm_grouped_wgrad_multi(int accumulate, const void* const* a_list, const void* const* b_list,
                           const int* rows_list, const int32_t* seg_offsets, int R, int E, int M,
                           int N, void* out, int ldo, void* workspace, int max_ctas,
                           void* stream) {
  return hm_grouped_wgrad_multi_shifted(accumulate, a_list, b_list, rows_list, seg_offsets, R, E, M, N, out,
                                        ldo, nullptr, nullptr, 0, workspace, max_ctas, stream);
}

int hm_grouped_wgrad_multi_shifted(int accumulate, const void* const* a_list, const void* const* b_list,
                                   const int* rows_list, const int32_t* seg_offsets, int R, int E, int M,
                                   int N, void* out, int ldo, const int32_t* shift_a,
                                   const int32_t* shift_b, int shift_stride, void* workspace,
                                   int max_ctas, void* stream) {
  if (R < 1 || R > hm::kMaxSegs) return fail(HM_E_SHAPE, "wgrad_multi: R=%d out of [1,%d]", R, hm::kMaxSegs);
  if (E < 1 || E > hm::kMaxExperts) return fail(HM_E_SHAPE, "wgrad_multi: E=%d out of range", E);
  if (M <= 0 || M % 8 || N <= 0 || N % 8 || ldo % 8) return fail(HM_E_SHAPE, "wgrad_multi: bad M/N/ldo");
  if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 127u))
    return fail(HM_E_ARG, "wgrad_multi: needs a 128-byte aligned workspace");
  cudaStream_t st = S(stream);
  hm::SegBases bases{};
  for (int j = 0; j < R; ++j) {
    if (!aligned16(a_list[j]) || !aligned16(b_list[j])) return fail(HM_E_ALIGN, "wgrad_multi: alignment");
    bases.a[j] = static_cast<const uint8_t*>(a_list[j]);
    bases.b[j] = static_cast<const uint8_t*>(b_list[j]);
  }
  const int rows0 = rows_list[0] > 0 ? rows_list[0] : 1;
  CUtensorMap ma, mb;
  uint64_t dims_a[2] = {(uint64_t)M, (uint64_t)rows0};
  uint64_t str_a[1] = {(uint64_t)M * 2};
  uint32_t box[2] = {64, 64};
  if (int rc = make_map(&ma, a_list[0], 2, dims_a, str_a, box)) return rc;
  uint64_t dims_b[2] = {(uint64_t)N, (uint64_t)rows0};
  uint64_t str_b[1] = {(uint64_t)N * 2};
  if (int rc = make_map(&mb, b_list[0], 2, dims_b, str_b, box)) return rc;
  CUtensorMap* maps = static_cast<CUtensorMap*>(workspace);
  hm::build_expert_maps_kernel<<<(E * R + 127) / 128, 128, 0, st>>>(
      ma, mb, seg_offsets, E, R, bases, static_cast<long>(M) * 2, static_cast<long>(N) * 2, maps, shift_a,
      shift_b, shift_stride);
  if (int rc = check_launch("build_expert_maps")) return rc;
  hm::GroupedGemmParams p{};
  p.seg_offsets = seg_offsets;  // segment 0 row table doubles as the GROUP_M bookkeeping
  p.R = R;
  p.E = E;
  p.M = M;
  p.N = N;
  p.out = static_cast<__nv_bfloat16*>(out);
  p.out_f32 = static_cast<float*>(out);
  p.ldo = ldo;
  p.expert_maps = maps;
  p.out_elems = static_cast<long>(E) * M * ldo;
  const TileBound tb{true, 0, M, N, E};
  if (accumulate)
    return launch_kind<true, true, true, hm::EPI_ACC_F32>(HM_GEMM_WGRAD_ACC, ma, mb, p, tb, max_ctas, st);
  return launch_kind<true, true, true, hm::EPI_STORE>(HM_GEMM_WGRAD, ma, mb, p, tb, max_ctas, st);
}

int hm_grouped_ffn_fwd(const void* x_perm, int rows, const int32_t* seg_offsets, int E,
                       const void* w_ug, const void* w_d, int d, int f, void* h, void* act,
                       void* y_perm, int max_ctas, void* stream) {
  if (f % 128 != 0) return fail(HM_E_SHAPE, "ffn: f=%d must be a multiple of 128", f);
  if (int rc = hm_grouped_gemm(HM_GEMM_FWD_UPGATE, x_perm, w_ug, seg_offsets, E, rows, 0, 2 * f, d,
                               act, f, h, 2 * f, nullptr, 0, nullptr, max_ctas, stream))
    return rc;
  return hm_grouped_gemm(HM_GEMM_FWD_DOWN, act, w_d, seg_offsets, E, rows, 0, d, f, y_perm, d,
                         nullptr, 0, nullptr, 0, nullptr, max_ctas, stream);
}

int hm_grouped_ffn_bwd(const void* dy_perm, const void* x_perm, const void* h, const void* act,
                       int rows, const int32_t* seg_offsets, int E, const void* w_ug,
                       const void* w_d, int d, int f, void* dh, void* dx_perm, void* dw_ug,
                       void* dw_d, void* workspace, int max_ctas, void* stream) {
  if (f % 128 != 0) return fail(HM_E_SHAPE, "ffn: f=%d must be a multiple of 128", f);
  // dH = SwiGLU'(dY . W_d[e]) : K = d, N = f
  if (int rc = hm_grouped_gemm(HM_GEMM_BWD_DACT, dy_perm, w_d, seg_offsets, E, rows, 0, f, d, dh,
                               2 * f, nullptr, 0, h, 2 * f, nullptr, max_ctas, stream))
    return rc;
  // dX = dH . W_ug[e] : K = 2f, N = d
  if (int rc = hm_grouped_gemm(HM_GEMM_BWD_DX, dh, w_ug, seg_offsets, E, rows, 0, d, 2 * f, dx_perm,
                               d, nullptr, 0, nullptr, 0, nullptr, max_ctas, stream))
    return rc;
  // dW_ug[e] = dH_e^T . X_e : M = 2f, N = d
  if (int rc = hm_grouped_gemm(HM_GEMM_WGRAD, dh, x_perm, seg_offsets, E, rows, 2 * f, d, 0, dw_ug,
                               d, nullptr, 0, nullptr, 0, workspace, max_ctas, stream))
    return rc;
  // dW_d[e] = dY_e^T . act_e : M = d, N = f  (second half of the workspace: the first call's
  // maps may still be in use by its kernel)
  return hm_grouped_gemm(HM_GEMM_WGRAD, dy_perm, act, seg_offsets, E, rows, d, f, 0, dw_d, f,
                         nullptr, 0, nullptr, 0,
                         static_cast<uint8_t*>(workspace) + hm_grouped_gemm_workspace_bytes(HM_GEMM_WGRAD, E),
                         max_ctas, stream);
}

}  // extern "C"
