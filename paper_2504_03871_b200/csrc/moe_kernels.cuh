// moe_kernels.cuh — K1 router/top-k, K2 dispatch permute (+ unpermute), K4 combine (+ bwd).
//
// Semantics fixed by the CPU oracle (oracle/moe_oracle.py, oracle/router_ref.c):
//  * router logits l[t,e] = sum_i x[t,i] * Wg[i,e] in fp32 with a FIXED "blocked" order. d is
//    split into blocks of 256 (j = 0 .. d/256-1). Inside block j, lane L of 32 accumulates
//    i = 256*j + 8*L + q for q = 0..7 with fused multiply-adds starting from 0 (bf16*bf16
//    products are exact in fp32, so FMA == mul-then-add), then the 32 lane partials are combined
//    by an xor butterfly (offsets 16, 8, 4, 2, 1) into the block partial P_j; finally
//    l = ((P_0 + P_1) + P_2) + ... in block order. Indices, counts and the permutation
//    therefore reproduce bit-for-bit on the CPU.
//  * an optional per-expert bias is added last (one fp32 rounding): l[t,e] = dot + bias[e]
//    (router skew for the Asym-EA sweep; bias-based load balancing).
//  * top-k: k largest logits, ties -> lower expert id, NaN after every number, each expert at
//    most once; w = softmax over the k selected logits.
//  * dispatch order: stable by (expert, token); a token appears at most once per expert.
//    Tokens are processed in chunks of kChunk; chunk c's rows for expert e start at
//    chunk_base[c][e] = offsets[e] + sum_{c'<c} count[c'][e].
#pragma once

#include "hm_common.cuh"

namespace hm {

constexpr int kChunk = 64;          // tokens per dispatch chunk (one permute CTA)
constexpr int kMaxTopK = 8;

// Top-k marks an already-selected expert with NaN: the comparator (v > best, or v == best with a
// lower id) never picks a NaN, so a selected expert cannot be chosen again even when the row's
// remaining logits are all -inf (a -inf mark would tie with the -inf start value and win on its
// lower id). When every unselected logit is NaN the fallback takes the lowest UNSELECTED id.
// Net rule (oracle/router_ref.c, moe_oracle.topk_softmax): rank by (isnan, -logit, expert id).
#define kSelectedMark __int_as_float(0x7fc00000)

// ------------------------------------------------------------------------------------------
// K1a: router logits (+ fused top-k, softmax, chunk histogram and scan when the experts form one
// group). Persistent: one CTA per SM (per expert group), each over a contiguous token range.
// Warp specialised: warps 0..15 compute, warps 16..19 are epilogue + producer (a rotating epilogue
// run by the compute warps themselves measured 1.6x slower: its top-k stalls the whole stage).
//  * token rows stream into a 4-stage shared-memory ring by 1-D bulk copies (TMA engine; 32 KB
//    stages of TG = 64 / nj tokens, nj = d / 256 blocks), issued by the epilogue that frees the slot;
//  * the router weight never touches shared memory: compute warp w owns block(s) j and keeps
//    Wg[256 j + 8 L + q, e0 .. e0 + EGW) in registers (lane L, q = 0..7: 8 x EGW fp32, in a
//    lane-dependent XOR order of the experts). Per (token, block) item a lane does 8 x EGW FMAs
//    (packed FFMA2: two IEEE fma.rn per instruction, the scalar per-accumulator sequence); the
//    warp reduces its EGW lane partials with a select-free reduce-scatter butterfly (offsets
//    16, 8, ... halving the vector, then plain xor steps: 9 shuffles for EGW = 8 instead of 40 —
//    and, fp32 addition being commutative, every expert's value is the full butterfly's tree);
//    two items are reduced together so their shuffle latencies overlap; block partials go to a
//    4-deep shared-memory table ring;
//  * epilogue warp 16 + s % 4 adds stage s's block partials in block order (+ bias) into logits,
//    runs the top-k / softmax on the logits still in registers as lane-parallel butterfly
//    argmaxes (FUSE), counts the chunk histogram with atomics, and refills the ring slot the
//    compute warps just released.
// mbarriers: full[slot] (bytes landed), pfull[slot] (16 compute warps wrote partial table slot),
// pempty[slot] (its epilogue warp consumed it). The last CTA to finish scans the per-chunk
// counts (FUSE).
constexpr int kRouterWarps = 16;     // compute warps
constexpr int kRouterEpiWarps = 4;   // epilogue warps: 20 warps take the register budget of 17
constexpr int kRouterThreads = (kRouterWarps + kRouterEpiWarps) * 32;
constexpr int kRouterStages = 4;     // ring slots == partial tables == epilogue warps
constexpr int kRouterNI = 2;         // items reduced together (shuffle ILP within 96 registers)
constexpr int kRouterStageBytes = 32768;  // 64 (token, block) items of 512 bytes
constexpr int kRouterItems = 64;

// Reduce-scatter butterfly of EGW values for NI items at once (shuffles interleaved). The values
// are in the lane's XOR-permuted expert order (slot r = expert r ^ router_lane_expert(lane);
// router_permute_slots), so at every halving level a lane keeps its low half and sends its high
// half with no selects: its partner (lane ^ off) holds the same experts in the opposite halves.
// Returns in out[i] the value of expert router_lane_expert<EGW>(lane) of item i, identical on
// the 32 / EGW lanes that share it.
template <int EGW, int NI>
HM_DEV void router_reduce_scatter(float (&v)[NI][EGW], float (&out)[NI]) {
  // the adds run as packed fp32x2 (FADD2: two IEEE adds per instruction, the same values):
  // adjacent slots of one item while a level keeps >= 2 values, else the NI items' values paired
  int off = 16;
#pragma unroll
  for (int h = EGW / 2; h >= 1; h >>= 1) {
    float r[NI][EGW / 2];
#pragma unroll
    for (int m = 0; m < h; ++m)
#pragma unroll
      for (int i = 0; i < NI; ++i) r[i][m] = __shfl_xor_sync(0xffffffffu, v[i][m + h], off);
    if (h >= 2) {
#pragma unroll
      for (int i = 0; i < NI; ++i)
#pragma unroll
        for (int m = 0; m < h; m += 2) {
          const float2 a = __fadd2_rn(make_float2(v[i][m], v[i][m + 1]), make_float2(r[i][m], r[i][m + 1]));
          v[i][m] = a.x;
          v[i][m + 1] = a.y;
        }
    } else {
#pragma unroll
      for (int i = 0; i + 1 < NI; i += 2) {
        const float2 a = __fadd2_rn(make_float2(v[i][0], v[i + 1][0]), make_float2(r[i][0], r[i + 1][0]));
        v[i][0] = a.x;
        v[i + 1][0] = a.y;
      }
      if (NI & 1) v[NI - 1][0] = v[NI - 1][0] + r[NI - 1][0];
    }
    off >>= 1;
  }
#pragma unroll
  for (int i = 0; i < NI; ++i) out[i] = v[i][0];
#pragma unroll
  for (int o = 32 / EGW / 2; o >= 1; o >>= 1) {
    float r[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) r[i] = __shfl_xor_sync(0xffffffffu, out[i], o);
#pragma unroll
    for (int i = 0; i + 1 < NI; i += 2) {
      const float2 a = __fadd2_rn(make_float2(out[i], out[i + 1]), make_float2(r[i], r[i + 1]));
      out[i] = a.x;
      out[i + 1] = a.y;
    }
    if (NI & 1) out[NI - 1] = out[NI - 1] + r[NI - 1];
  }
}

// Natural expert order -> the lane's XOR-permuted order (slot r <- expert r ^ mask, mask =
// router_lane_expert(lane)): one conditional half swap per halving level.
template <int EGW>
HM_DEV void router_permute_slots(float (&w)[EGW], int lane) {
  int off = 16;
#pragma unroll
  for (int h = EGW / 2; h >= 1; h >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int m = 0; m < EGW; ++m)
      if ((m & h) == 0) {
        const float a = w[m], c = w[m + h];
        w[m] = up ? c : a;
        w[m + h] = up ? a : c;
      }
    off >>= 1;
  }
}

template <int EGW>
HM_DEV int router_lane_expert(int lane) {
  int e = 0, off = 16;
#pragma unroll
  for (int h = EGW / 2; h >= 1; h >>= 1) {
    if (lane & off) e += h;
    off >>= 1;
  }
  return e;
}

// Per-expert totals, exclusive offsets and per-chunk row bases (in place) from per-chunk counts.
// Threads (g, e) of the CTA: chunk group g of G = blockDim / Epad, expert e; loads coalesced
// over e. part: blockDim ints of shared memory, off: 257 ints.
HM_DEV void router_scan_block(int32_t* __restrict__ chunk_counts /*in: counts, out: bases*/, int nchunk,
                              int E, int32_t* __restrict__ counts, int32_t* __restrict__ offsets,
                              int* part, int* off) {
  int epad = 1;
  while (epad < E) epad <<= 1;
  const int G = blockDim.x / epad;
  const int g = threadIdx.x / epad, e = threadIdx.x % epad;
  const int c_lo = static_cast<int>((static_cast<long>(nchunk) * g) / G);
  const int c_hi = static_cast<int>((static_cast<long>(nchunk) * (g + 1)) / G);
  int s = 0;
  if (e < E && g < G) {
#pragma unroll 8
    for (int c = c_lo; c < c_hi; ++c) s += __ldcg(chunk_counts + static_cast<long>(c) * E + e);
  }
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x < epad) {  // exclusive prefix over the chunk groups of expert e = threadIdx.x
    int a = 0;
    for (int gg = 0; gg < G; ++gg) {
      const int v = part[gg * epad + threadIdx.x];
      part[gg * epad + threadIdx.x] = a;
      a += v;
    }
    if (threadIdx.x < E) off[threadIdx.x] = a;  // expert total, scanned below
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0;
    for (int i = 0; i < E; ++i) {
      const int t = off[i];
      off[i] = a;
      counts[i] = t;
      offsets[i] = a;
      a += t;
    }
    off[E] = a;
    offsets[E] = a;
  }
  __syncthreads();
  if (e < E && g < G) {
    int base = off[e] + part[threadIdx.x];
#pragma unroll 8
    for (int c = c_lo; c < c_hi; ++c) {
      int32_t* p = chunk_counts + static_cast<long>(c) * E + e;
      const int v = __ldcg(p);
      *p = base;
      base += v;
    }
  }
}

// HM_ROUTER_TIMELINE builds: per-CTA globaltimer stamps (ns) of the fused router's phases,
// [cta][0] entry, [1] weights in registers (after the first CTA barrier), [2] last compute stage
// done (compute warp 0), [3] last epilogue stage done (epilogue warp 16), [4] CTA exit; [511][0..1]
// the last CTA's scan begin / end. Read by hm_debug_router_timeline (tools/router_timeline.py).
__device__ unsigned long long g_router_tl[512][5];
HM_DEV unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#ifdef HM_ROUTER_TIMELINE
#define HM_RT_STAMP(i) g_router_tl[blockIdx.x][i] = globaltimer_ns()
#else
#define HM_RT_STAMP(i) do { } while (0)
#endif

struct RouterShared {
  uint64_t full[kRouterStages];
  uint64_t pfull[kRouterStages];
  uint64_t pempty[kRouterStages];
  int is_last;
  int scan_off[257];
};

// Top-k of one token whose EGW logits sit in EGW consecutive lanes (lane e of the group holds
// expert e; e >= E is no expert): k rounds of a lexicographic (value desc, id asc) butterfly
// argmax over the group with NaN never eligible — the comparator of the sequential scan
// (router_topk_lane_kernel), so the same experts in the same order — the winner marked NaN, the
// all-NaN fallback to the lowest unselected id; then the softmax over the selected logits
// (sequential sum in slot order). Lane e == s writes slot s and counts it in the histogram.
template <int EGW>
HM_DEV void router_select_lanes(float v, int e, int E, int k, bool write, int32_t* idx_out, float* w_out,
                                int32_t* hist_row) {
  float cur = (e < E) ? v : kSelectedMark;
  float sel_l[kMaxTopK];
  int sel_e[kMaxTopK];
  unsigned taken = 0u;
#pragma unroll
  for (int s = 0; s < kMaxTopK; ++s) {
    if (s < k) {
      const bool ok = (e < E) && !isnan(cur);
      float bv = ok ? cur : -INFINITY;
      int be = ok ? e : 0x7fffffff;
#pragma unroll
      for (int off = 1; off < EGW; off <<= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int oe = __shfl_xor_sync(0xffffffffu, be, off);
        if (ov > bv || (ov == bv && oe < be)) { bv = ov; be = oe; }
      }
      if (be == 0x7fffffff) {  // every unselected logit is NaN: lowest unselected id
        be = __ffs(~taken) - 1;
        bv = kSelectedMark;
      }
      taken |= 1u << be;
      sel_l[s] = bv;
      sel_e[s] = be;
      if (e == be) cur = kSelectedMark;
    }
  }
  float ex[kMaxTopK];
  float sum = 0.f;
#pragma unroll
  for (int s = 0; s < kMaxTopK; ++s)
    if (s < k) { ex[s] = expf(sel_l[s] - sel_l[0]); sum += ex[s]; }
#pragma unroll
  for (int s = 0; s < kMaxTopK; ++s)
    if (s < k && e == s && write) {
      idx_out[s] = sel_e[s];
      w_out[s] = ex[s] / sum;
      atomicAdd(hist_row + sel_e[s], 1);
    }
}

// EGW experts per CTA group held by every compute warp (registers: BPW * 8 * EGW <= 64 floats),
// nj = d / 256 blocks: a template constant for the powers of two (every index a shift), else
// NJ_T = 0 and nj = d / 256 at run time (any d % 256 == 0 up to 16384). Warp -> work map:
//   nj <= 16: P = 16 / nj token streams; warp w < P * nj owns block w % nj and tokens
//             w / nj + P * m (m = 0..3) of each stage of TG = 4 P tokens (idle warps: 16 % nj);
//   nj > 16:  BPW = ceil(nj / 16) blocks per warp (w + 16 b), every token of a TG = 4 / BPW stage.
// FUSE: one expert group (E <= EGW): top-k, softmax, the per-chunk histogram (atomics into the
// zeroed chunk_counts) and, in the last CTA, the scan.
// the epilogue warp that handles the CTA's last stage (stage nst - 1 goes to warp (nst-1) % 4)
HM_DEV bool s_last_epi(int nst, int epi) { return nst > 0 && (nst - 1) % kRouterEpiWarps == epi; }

template <int EGW, int NJ_T, int BPW, bool FUSE>
__global__ void __launch_bounds__(kRouterThreads, 1)
    router_fused_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wg,
                        const float* __restrict__ bias, int T, int d_arg, int E, int ranges,
                        float* __restrict__ logits, int k, int32_t* __restrict__ idx,
                        float* __restrict__ w, int32_t* __restrict__ chunk_counts /*[nchunk*E + 1]*/,
                        int32_t* __restrict__ counts, int32_t* __restrict__ offsets) {
  static_assert(BPW * 8 * EGW <= 64, "router weights per thread");
  const int nj = NJ_T > 0 ? NJ_T : (d_arg >> 8);
  const int P = nj <= 16 ? 16 / nj : 1;        // token streams (nj <= 16)
  const int TG = nj <= 16 ? 4 * P : 4 / BPW;   // tokens per stage
  const int D = nj * 256;
  const long kRowBytes = static_cast<long>(D) * 2;
  const int kRounds = (TG * EGW + 31) / 32;    // epilogue lane rounds per stage
  extern __shared__ __align__(1024) uint8_t smem_rt[];
  uint8_t* ring = smem_rt;                                                  // stages x 32 KB
  float* part = reinterpret_cast<float*>(smem_rt + kRouterStages * kRouterStageBytes);  // [4][64][EGW]
  RouterShared& sh = *reinterpret_cast<RouterShared*>(part + kRouterStages * kRouterItems * EGW);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int groups = gridDim.x / ranges;
  const int group = blockIdx.x % groups;
  const int range = blockIdx.x / groups;
  const int e0 = group * EGW;
  const long units = (T + TG - 1) / TG;
  const int t_begin = static_cast<int>(units * range / ranges) * TG;
  const int t_end = min(T, static_cast<int>(units * (range + 1) / ranges) * TG);
  const int nst = t_end > t_begin ? (t_end - t_begin + TG - 1) / TG : 0;

  if (threadIdx.x == 0) {
    HM_RT_STAMP(0);
    for (int s = 0; s < kRouterStages; ++s) {
      mbar_init(&sh.full[s], 1);
      mbar_init(&sh.pfull[s], kRouterWarps);
      mbar_init(&sh.pempty[s], 1);
    }
    fence_barrier_init();
    for (int s = 0; s < kRouterStages && s < nst; ++s) {
      const int t0 = t_begin + s * TG;
      const uint32_t bytes = static_cast<uint32_t>(min(TG, t_end - t0) * kRowBytes);
      mbar_arrive_expect_tx(&sh.full[s], bytes);
      bulk_load_1d(ring + s * kRouterStageBytes, x + static_cast<long>(t0) * D, bytes, &sh.full[s]);
    }
  }
  // this warp's blocks and items (warp-uniform validity)
  const bool active = warp < kRouterWarps && (nj > 16 || warp < P * nj);
  int jb[BPW];
#pragma unroll
  for (int b = 0; b < BPW; ++b) jb[b] = (nj <= 16) ? (warp % nj) : (warp + 16 * b);
  float wr[BPW][8][EGW];
  const uint16_t* wg16 = reinterpret_cast<const uint16_t*>(wg);
#pragma unroll
  for (int b = 0; b < BPW; ++b)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const long i = 256L * jb[b] + 8 * lane + q;
      if (!active || jb[b] >= nj) {  // epilogue / idle warps and missing blocks hold no weights
#pragma unroll
        for (int e = 0; e < EGW; ++e) wr[b][q][e] = 0.f;
      } else if (E % EGW == 0) {  // the group's EGW weights of row i are one aligned vector
        uint32_t u[EGW / 2];
        if (EGW == 8) {
          const uint4 t = __ldg(reinterpret_cast<const uint4*>(wg16 + i * E + e0));
          u[0] = t.x; u[1 % (EGW / 2)] = t.y; u[2 % (EGW / 2)] = t.z; u[3 % (EGW / 2)] = t.w;
        } else if (EGW == 4) {
          const uint2 t = __ldg(reinterpret_cast<const uint2*>(wg16 + i * E + e0));
          u[0] = t.x; u[1 % (EGW / 2)] = t.y;
        } else {
          u[0] = __ldg(reinterpret_cast<const uint32_t*>(wg16 + i * E + e0));
        }
#pragma unroll
        for (int e = 0; e < EGW; e += 2) {
          wr[b][q][e] = __uint_as_float(u[e / 2] << 16);
          wr[b][q][e + 1] = __uint_as_float(u[e / 2] & 0xffff0000u);
        }
      } else {
#pragma unroll
        for (int e = 0; e < EGW; ++e) wr[b][q][e] = (e0 + e < E) ? bf16_to_f32(wg16[i * E + e0 + e]) : 0.f;
      }
      router_permute_slots<EGW>(wr[b][q], lane);
    }
  const int my_e = router_lane_expert<EGW>(lane);
  const bool writer = (lane & (32 / EGW - 1)) == 0;
  int ti_of[4], xoff[4], poff[4];
  bool item_ok[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int b = (nj <= 16) ? 0 : m % BPW;
    ti_of[m] = (nj <= 16) ? warp / nj + P * m : m / BPW;
    item_ok[m] = active && jb[b] < nj && ti_of[m] < TG;
    xoff[m] = item_ok[m] ? static_cast<int>(ti_of[m] * kRowBytes + (256 * jb[b] + 8 * lane) * 2) : 0;
    poff[m] = (ti_of[m] * nj + jb[b]) * EGW + my_e;
  }
  // a lane's expert in the epilogue is lane % EGW in every round (32 % EGW == 0)
  const float bias_lane = (bias && e0 + lane % EGW < E) ? bias[e0 + lane % EGW] : 0.f;
  __syncthreads();
  if (threadIdx.x == 0) HM_RT_STAMP(1);

  if (warp < kRouterWarps) {
    // ============ compute warps ============
    for (int s = 0; s < nst; ++s) {
      const int slot = s % kRouterStages;
      const int nt = min(TG, t_end - (t_begin + s * TG));
      float* pb = part + slot * kRouterItems * EGW;
      mbar_wait(&sh.full[slot], (s / kRouterStages) & 1);
      if (s >= kRouterStages) mbar_wait(&sh.pempty[slot], ((s / kRouterStages) - 1) & 1);
      const uint8_t* st = ring + slot * kRouterStageBytes;
      if (active) {
        float acc[kRouterNI][EGW];
#pragma unroll
        for (int m0 = 0; m0 < 4; m0 += kRouterNI) {
          if (!item_ok[m0]) continue;  // warp-uniform; items of a pair are both valid or the
                                       // second is masked below
#pragma unroll
          for (int u = 0; u < kRouterNI; ++u) {
            const int m = m0 + u;
            const int b = (nj <= 16) ? 0 : m % BPW;
            // a token past the stage's end reads stale ring bytes; its result is never stored
            const uint4 xv = item_ok[m] ? *reinterpret_cast<const uint4*>(st + xoff[m]) : make_uint4(0u, 0u, 0u, 0u);
            const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
            for (int e = 0; e < EGW; ++e) acc[u][e] = 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float xf = __uint_as_float((q & 1) ? (xw[q >> 1] & 0xffff0000u) : (xw[q >> 1] << 16));
#pragma unroll
              for (int e = 0; e < EGW; e += 2) {
                const float2 r = __ffma2_rn(make_float2(xf, xf), make_float2(wr[b][q][e], wr[b][q][e + 1]),
                                            make_float2(acc[u][e], acc[u][e + 1]));
                acc[u][e] = r.x;
                acc[u][e + 1] = r.y;
              }
            }
          }
          float pj[kRouterNI];
          router_reduce_scatter<EGW, kRouterNI>(acc, pj);
#pragma unroll
          for (int u = 0; u < kRouterNI; ++u)
            if (writer && item_ok[m0 + u] && ti_of[m0 + u] < nt) pb[poff[m0 + u]] = pj[u];
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.pfull[slot]);  // releases this warp's ring reads and table writes
    }
    if (threadIdx.x == 0) HM_RT_STAMP(2);
  } else {
    // ============ epilogue warps: stage s is warp 16 + s % 4's; it refills ring slot s % 4 ============
    for (int s = warp - kRouterWarps; s < nst; s += kRouterEpiWarps) {
      const int slot = s % kRouterStages;
      const int t0 = t_begin + s * TG;
      const int nt = min(TG, t_end - t0);
      const float* pb = part + slot * kRouterItems * EGW;
      mbar_wait(&sh.pfull[slot], (s / kRouterStages) & 1);
      if (lane == 0 && s + kRouterStages < nst) {  // every compute warp is done with this slot
        const int tn = t_begin + (s + kRouterStages) * TG;
        const uint32_t bytes = static_cast<uint32_t>(min(TG, t_end - tn) * kRowBytes);
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&sh.full[slot], bytes);
        bulk_load_1d(ring + slot * kRouterStageBytes, x + static_cast<long>(tn) * D, bytes, &sh.full[slot]);
      }
      // block partials -> logits in block order (+ bias): lane (ti, e), e fastest
      for (int r = 0; r < kRounds; ++r) {
        const int id = r * 32 + lane;
        const int ti = id / EGW, e = id % EGW;
        const int tl = id < TG * EGW ? ti : 0;  // lanes past the stage's items read item 0
        float v;
        if (NJ_T > 0) {
          constexpr int NJC = NJ_T > 0 ? NJ_T : 1;
          float pv[NJC];
#pragma unroll
          for (int j = 0; j < NJC; ++j) pv[j] = pb[(tl * NJC + j) * EGW + e];
          v = pv[0];
#pragma unroll
          for (int j = 1; j < NJC; ++j) v = v + pv[j];
        } else {
          v = pb[(tl * nj) * EGW + e];
          for (int j = 1; j < nj; ++j) v = v + pb[(tl * nj + j) * EGW + e];
        }
        if (bias) v = v + bias_lane;
        const bool ok = id < TG * EGW && ti < nt;
        if (ok && e0 + e < E) logits[static_cast<long>(t0 + ti) * E + e0 + e] = v;
        if (FUSE) {
          const long t = t0 + (ok ? ti : 0);
          router_select_lanes<EGW>(v, e, E, k, ok, idx + t * k, w + t * k, chunk_counts + (t / kChunk) * E);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.pempty[slot]);
    }
    if (lane == 0 && s_last_epi(nst, warp - kRouterWarps)) HM_RT_STAMP(3);
  }
  if (FUSE) {
    // the last CTA to finish turns the per-chunk counts into totals, offsets and chunk bases
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const int nchunk = (T + kChunk - 1) / kChunk;
      const int prev = atomicAdd(chunk_counts + static_cast<long>(nchunk) * E, 1);
      sh.is_last = (prev == static_cast<int>(gridDim.x) - 1);
    }
    __syncthreads();
    if (sh.is_last) {
      __threadfence();
#ifdef HM_ROUTER_TIMELINE
      if (threadIdx.x == 0) g_router_tl[511][0] = globaltimer_ns();
#endif
      const int nchunk = (T + kChunk - 1) / kChunk;
      router_scan_block(chunk_counts, nchunk, E, counts, offsets, reinterpret_cast<int*>(ring), sh.scan_off);
#ifdef HM_ROUTER_TIMELINE
      __syncthreads();
      if (threadIdx.x == 0) g_router_tl[511][1] = globaltimer_ns();
#endif
    }
  }
  if (threadIdx.x == 0) HM_RT_STAMP(4);
}

constexpr size_t router_fused_smem_bytes(int egw) {
  return static_cast<size_t>(kRouterStages) * kRouterStageBytes + kRouterStages * kRouterItems * egw * 4 +
         sizeof(RouterShared) + 16;
}

// ------------------------------------------------------------------------------------------
// K1b: top-k + softmax + per-chunk expert histogram. One CTA per chunk of kChunk tokens,
// one warp per token (looping). E <= 256.
__global__ void __launch_bounds__(1024)
    router_topk_kernel(const float* __restrict__ logits, int T, int E, int k,
                       int32_t* __restrict__ idx, float* __restrict__ w,
                       int32_t* __restrict__ chunk_counts /*[nchunk][E]*/) {
  __shared__ int hist[256];
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist[e] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x;
  const int tbeg = c * kChunk, tend = min(T, tbeg + kChunk);
  constexpr int kPer = 8;  // values per lane (E <= 256)
  const int nwarps = blockDim.x >> 5;
  for (int t = tbeg + warp; t < tend; t += nwarps) {
    float v[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int e = q * 32 + lane;
      v[q] = (e < E) ? logits[static_cast<long>(t) * E + e] : -INFINITY;
    }
    float sel_l[kMaxTopK];
    int sel_e[kMaxTopK];
    for (int s = 0; s < k; ++s) {
      // lane-local best (ties -> lower id = lower q since e = q*32+lane ascends with q)
      float bv = -INFINITY;
      int be = 0x7fffffff;
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int e = q * 32 + lane;
        if (e < E && (v[q] > bv || (v[q] == bv && e < be))) { bv = v[q]; be = e; }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int oe = __shfl_xor_sync(0xffffffffu, be, off);
        if (ov > bv || (ov == bv && oe < be)) { bv = ov; be = oe; }
      }
      if (be == 0x7fffffff) {
        // every remaining logit is NaN: take the lowest unselected expert so indices stay valid
        be = 0;
        bv = kSelectedMark;  // the selected logit is NaN (the softmax sees it)
        for (int p = 0; p < s; ++p)
          if (sel_e[p] == be) { ++be; p = -1; }
      }
      sel_l[s] = bv;
      sel_e[s] = be;
#pragma unroll
      for (int q = 0; q < kPer; ++q)
        if (q * 32 + lane == be) v[q] = kSelectedMark;
    }
    if (lane == 0) {
      // softmax over the k selected logits (sel_l[0] is the max)
      float ex[kMaxTopK];
      float sum = 0.f;
      for (int s = 0; s < k; ++s) { ex[s] = expf(sel_l[s] - sel_l[0]); sum += ex[s]; }
      for (int s = 0; s < k; ++s) {
        idx[static_cast<long>(t) * k + s] = sel_e[s];
        w[static_cast<long>(t) * k + s] = ex[s] / sum;
        atomicAdd(&hist[sel_e[s]], 1);
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    chunk_counts[static_cast<long>(c) * E + e] = hist[e];
}

// K1b (v2, E % 4 == 0, E <= EP <= 64): one THREAD per token, one CTA of kChunk threads per
// chunk. The token's E logits sit in registers (float4 loads); each of the k rounds scans them in
// ascending expert order with router_topk_kernel's comparator (v > best, or v == best with a
// lower id; NaN never wins). That comparator is a lexicographic max over the non-NaN values, so
// the sequential scan selects exactly what the warp butterfly selects, including the all-NaN
// fallback; softmax and histogram are the same code. No shuffles: C3 (E = 64, k = 6) spent
// 32 us in the warp-per-token kernel's 60 dependent shuffles per token.
template <int EP>
__global__ void __launch_bounds__(kChunk)
    router_topk_lane_kernel(const float* __restrict__ logits, int T, int E, int k,
                            int32_t* __restrict__ idx, float* __restrict__ w,
                            int32_t* __restrict__ chunk_counts /*[nchunk][E]*/) {
  __shared__ int hist[EP];
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist[e] = 0;
  __syncthreads();
  const int c = blockIdx.x;
  const int t = c * kChunk + threadIdx.x;
  if (t < T) {
    float v[EP];
#pragma unroll
    for (int q = 0; q < EP / 4; ++q) {
      float4 f = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      if (4 * q < E) f = __ldg(reinterpret_cast<const float4*>(logits + static_cast<long>(t) * E) + q);
      v[4 * q] = f.x; v[4 * q + 1] = f.y; v[4 * q + 2] = f.z; v[4 * q + 3] = f.w;
    }
    float sel_l[kMaxTopK];
    int sel_e[kMaxTopK];
    for (int s = 0; s < k; ++s) {
      float bv = -INFINITY;
      int be = 0x7fffffff;
#pragma unroll
      for (int e = 0; e < EP; ++e)
        if (e < E && (v[e] > bv || (v[e] == bv && e < be))) { bv = v[e]; be = e; }
      if (be == 0x7fffffff) {
        be = 0;
        bv = kSelectedMark;  // the selected logit is NaN (the softmax sees it)
        for (int p = 0; p < s; ++p)
          if (sel_e[p] == be) { ++be; p = -1; }
      }
      sel_l[s] = bv;
      sel_e[s] = be;
#pragma unroll
      for (int e = 0; e < EP; ++e)
        if (e == be) v[e] = kSelectedMark;
    }
    float ex[kMaxTopK];
    float sum = 0.f;
    for (int s = 0; s < k; ++s) { ex[s] = expf(sel_l[s] - sel_l[0]); sum += ex[s]; }
    for (int s = 0; s < k; ++s) {
      idx[static_cast<long>(t) * k + s] = sel_e[s];
      w[static_cast<long>(t) * k + s] = ex[s] / sum;
      atomicAdd(&hist[sel_e[s]], 1);
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    chunk_counts[static_cast<long>(c) * E + e] = hist[e];
}

// ------------------------------------------------------------------------------------------
// K1c: counts / offsets / chunk bases (the unfused router path). Single CTA of 1024 threads.
__global__ void __launch_bounds__(1024)
    router_scan_kernel(int32_t* __restrict__ chunk_counts /*in: counts, out: bases*/, int nchunk,
                       int E, int32_t* __restrict__ counts, int32_t* __restrict__ offsets) {
  __shared__ int part[1024];
  __shared__ int off[257];
  router_scan_block(chunk_counts, nchunk, E, counts, offsets, part, off);
}

// ------------------------------------------------------------------------------------------
// Stable destination rows of one chunk: warp w handles experts w, w+8, ...; for each expert it
// scans the chunk's (token, slot) entries 32 at a time with a ballot, so entry i of expert e
// gets row base[e] + #(earlier entries of e). Tokens hold distinct experts, so entry order ==
// token order within an expert.
HM_DEV void assign_rows_ballot(const int* s_idx, int* s_row, const int32_t* base, int n, int E) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  for (int e = warp; e < E; e += nwarps) {
    int r = base[e];
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      const bool hit = (i < n) && (s_idx[i] == e);
      const uint32_t m = __ballot_sync(0xffffffffu, hit);
      if (hit) s_row[i] = r + __popc(m & ((1u << lane) - 1u));
      r += __popc(m);
    }
  }
}

// ------------------------------------------------------------------------------------------
// K2: dispatch permute. One CTA per chunk: (1) thread e walks the chunk's tokens in order and
// assigns destination rows for expert e (stable), (2) warps copy token rows with 128-bit loads
// and k 128-bit stores per 16-byte segment.
template <int VPL>  // 16-byte vectors per lane per token row (d = VPL * 256)
__global__ void __launch_bounds__(256)
    dispatch_permute_kernel(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ idx,
                            const int32_t* __restrict__ chunk_base, int T, int d, int E, int k,
                            __nv_bfloat16* __restrict__ x_perm, int32_t* __restrict__ row_src,
                            int32_t* __restrict__ row_of) {
  __shared__ int s_idx[kChunk * kMaxTopK];
  __shared__ int s_row[kChunk * kMaxTopK];
  const int c = blockIdx.x;
  const int tbeg = c * kChunk;
  const int nt = min(kChunk, T - tbeg);
  for (int i = threadIdx.x; i < nt * k; i += blockDim.x) s_idx[i] = idx[static_cast<long>(tbeg) * k + i];
  __syncthreads();
  assign_rows_ballot(s_idx, s_row, chunk_base + static_cast<long>(c) * E, nt * k, E);
  __syncthreads();
  if (blockIdx.y == 0) {
    for (int i = threadIdx.x; i < nt * k; i += blockDim.x) {
      const int r = s_row[i];
      row_of[static_cast<long>(tbeg) * k + i] = r;
      row_src[r] = tbeg + i / k;
    }
  }
  // row copies; with gridDim.y = S > 1 the S CTAs of a chunk (each re-deriving the chunk's
  // rows, a few hundred shared-memory operations) copy every S-th group of 8 tokens
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int tt = warp + 8 * blockIdx.y; tt < nt; tt += 8 * gridDim.y) {
    const long t = tbeg + tt;
    const uint4* src = reinterpret_cast<const uint4*>(x + t * d);
    uint4 v[VPL];
#pragma unroll
    for (int q = 0; q < VPL; ++q) v[q] = __ldg(src + q * 32 + lane);
    for (int s = 0; s < k; ++s) {
      uint4* dst = reinterpret_cast<uint4*>(x_perm + static_cast<long>(s_row[tt * k + s]) * d);
#pragma unroll
      for (int q = 0; q < VPL; ++q) dst[q * 32 + lane] = v[q];
    }
  }
}

// generic-d fallback of the row copy (d multiple of 8)
__global__ void __launch_bounds__(256)
    dispatch_permute_generic_kernel(const __nv_bfloat16* __restrict__ x,
                                    const int32_t* __restrict__ idx,
                                    const int32_t* __restrict__ chunk_base, int T, int d, int E,
                                    int k, __nv_bfloat16* __restrict__ x_perm,
                                    int32_t* __restrict__ row_src, int32_t* __restrict__ row_of) {
  __shared__ int s_idx[kChunk * kMaxTopK];
  __shared__ int s_row[kChunk * kMaxTopK];
  const int c = blockIdx.x;
  const int tbeg = c * kChunk;
  const int nt = min(kChunk, T - tbeg);
  for (int i = threadIdx.x; i < nt * k; i += blockDim.x) s_idx[i] = idx[static_cast<long>(tbeg) * k + i];
  __syncthreads();
  assign_rows_ballot(s_idx, s_row, chunk_base + static_cast<long>(c) * E, nt * k, E);
  __syncthreads();
  for (int i = threadIdx.x; i < nt * k; i += blockDim.x) {
    const int r = s_row[i];
    row_of[static_cast<long>(tbeg) * k + i] = r;
    row_src[r] = tbeg + i / k;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nv = d / 8;
  for (int tt = warp; tt < nt; tt += 8) {
    const long t = tbeg + tt;
    const uint4* src = reinterpret_cast<const uint4*>(x + t * d);
    for (int q = lane; q < nv; q += 32) {
      const uint4 v = __ldg(src + q);
      for (int s = 0; s < k; ++s)
        reinterpret_cast<uint4*>(x_perm + static_cast<long>(s_row[tt * k + s]) * d)[q] = v;
    }
  }
}

// ------------------------------------------------------------------------------------------
// K4: combine. y[t] = sum_s w[t,s] * y_perm[row_of[t,s]] (fp32 accumulate in slot order).
// One warp per token; lane handles 8-element (16-byte) segments.
template <int K>
__global__ void __launch_bounds__(256)
    combine_kernel(const __nv_bfloat16* __restrict__ y_perm, const int32_t* __restrict__ row_of,
                   const float* __restrict__ w, int T, int d, __nv_bfloat16* __restrict__ y) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int nv = d / 8;
  for (int t = warp; t < T; t += nwarps) {
    int rows[kMaxTopK];
    float ws[kMaxTopK];
    for (int s = 0; s < K; ++s) {
      rows[s] = row_of[static_cast<long>(t) * K + s];
      ws[s] = w[static_cast<long>(t) * K + s];
    }
    // CU column segments per lane in flight before any is consumed (memory-level parallelism:
    // one segment per row at a time left the C2 combine at ~74 % of HBM; C3, k = 6: -3 %)
    constexpr int CU = K <= 2 ? 4 : 2;
    for (int q0 = lane; q0 < nv; q0 += 32 * CU) {
      uint4 v[CU][K];
#pragma unroll
      for (int u = 0; u < CU; ++u)
#pragma unroll
        for (int s = 0; s < K; ++s)
          if (q0 + 32 * u < nv)
            v[u][s] = __ldg(reinterpret_cast<const uint4*>(y_perm + static_cast<long>(rows[s]) * d) + q0 + 32 * u);
#pragma unroll
      for (int u = 0; u < CU; ++u) {
        const int q = q0 + 32 * u;
        if (q >= nv) break;
        float acc[8];
#pragma unroll
        for (int z = 0; z < 8; ++z) acc[z] = 0.f;
#pragma unroll
        for (int s = 0; s < K; ++s) {
          const uint16_t* h = reinterpret_cast<const uint16_t*>(&v[u][s]);
#pragma unroll
          for (int z = 0; z < 8; ++z) acc[z] = __fmaf_rn(ws[s], bf16_to_f32(h[z]), acc[z]);
        }
        uint4 o;
        o.x = pack_bf16x2(acc[0], acc[1]);
        o.y = pack_bf16x2(acc[2], acc[3]);
        o.z = pack_bf16x2(acc[4], acc[5]);
        o.w = pack_bf16x2(acc[6], acc[7]);
        reinterpret_cast<uint4*>(y + static_cast<long>(t) * d)[q] = o;
      }
    }
  }
}

// combine backward: dy_perm[row_of[t,s]] = w[t,s] * dy[t];  dw[t,s] = <dy[t], y_perm[row_of[t,s]]>
template <int K>
__global__ void __launch_bounds__(256)
    combine_bwd_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ y_perm,
                       const int32_t* __restrict__ row_of, const float* __restrict__ w, int T, int d, __nv_bfloat16* __restrict__ dy_perm, float* __restrict__ dw) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int nv = d / 8;
  for (int t = warp; t < T; t += nwarps) {
    int rows[kMaxTopK];
    float ws[kMaxTopK], dot[kMaxTopK];
    for (int s = 0; s < K; ++s) {
      rows[s] = row_of[static_cast<long>(t) * K + s];
      ws[s] = w[static_cast<long>(t) * K + s];
      dot[s] = 0.f;
    }
    // CU column segments per lane loaded before any is consumed (memory-level parallelism: C2
    // 0.116 -> 0.106 ms, C3 0.167 -> 0.141 ms); the segments are then consumed in column order,
    // so dw keeps its summation order
#ifndef HM_COMBINE_BWD_CU
#define HM_COMBINE_BWD_CU 4
#endif
    constexpr int CU = K <= 2 ? HM_COMBINE_BWD_CU : 2;
    for (int q0 = lane; q0 < nv; q0 += 32 * CU) {
      uint4 g[CU], yv[CU][K];
#pragma unroll
      for (int u = 0; u < CU; ++u)
        if (q0 + 32 * u < nv) {
          g[u] = __ldg(reinterpret_cast<const uint4*>(dy + static_cast<long>(t) * d) + q0 + 32 * u);
#pragma unroll
          for (int s = 0; s < K; ++s)
            yv[u][s] = __ldg(reinterpret_cast<const uint4*>(y_perm + static_cast<long>(rows[s]) * d) + q0 + 32 * u);
        }
#pragma unroll
      for (int u = 0; u < CU; ++u) {
        const int q = q0 + 32 * u;
        if (q >= nv) break;
        const uint16_t* gh = reinterpret_cast<const uint16_t*>(&g[u]);
        float gf[8];
#pragma unroll
        for (int z = 0; z < 8; ++z) gf[z] = bf16_to_f32(gh[z]);
#pragma unroll
        for (int s = 0; s < K; ++s) {
          const uint16_t* yh = reinterpret_cast<const uint16_t*>(&yv[u][s]);
#pragma unroll
          for (int z = 0; z < 8; ++z) dot[s] = __fmaf_rn(gf[z], bf16_to_f32(yh[z]), dot[s]);
          uint4 o;
          o.x = pack_bf16x2(ws[s] * gf[0], ws[s] * gf[1]);
          o.y = pack_bf16x2(ws[s] * gf[2], ws[s] * gf[3]);
          o.z = pack_bf16x2(ws[s] * gf[4], ws[s] * gf[5]);
          o.w = pack_bf16x2(ws[s] * gf[6], ws[s] * gf[7]);
          reinterpret_cast<uint4*>(dy_perm + static_cast<long>(rows[s]) * d)[q] = o;
        }
      }
    }
    for (int s = 0; s < K; ++s) {
      float v = dot[s];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) dw[static_cast<long>(t) * K + s] = v;
    }
  }
}

// ------------------------------------------------------------------------------------------
// Dispatch backward fused with the router's input gradient:
//   dlogit[t,s] = w[t,s] * (dw[t,s] - sum_j w[t,j] dw[t,j])        (softmax over the selected k)
//   dx[t]       = sum_s dx_perm[row_of[t,s]] + sum_s dlogit[t,s] * Wg[:, idx[t,s]]
// wg_t is Wg transposed ([E][d]). Also writes dlogit (for the router weight gradient).
template <int K>
__global__ void __launch_bounds__(256, 4)
    unpermute_router_bwd_kernel(const __nv_bfloat16* __restrict__ dx_perm,
                                const int32_t* __restrict__ row_of, const int32_t* __restrict__ idx,
                                const float* __restrict__ w, const float* __restrict__ dw,
                                const __nv_bfloat16* __restrict__ wg_t, int T, int d,
                                __nv_bfloat16* __restrict__ dx, float* __restrict__ dlogit,
                                float* __restrict__ dl_perm, float* __restrict__ coef8 = nullptr) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int nv = d / 8;
  for (int t = warp; t < T; t += nwarps) {
    int rows[kMaxTopK], ex[kMaxTopK];
    float dl[kMaxTopK];
    float wsum = 0.f;
    for (int s = 0; s < K; ++s) {
      rows[s] = row_of[static_cast<long>(t) * K + s];
      ex[s] = idx[static_cast<long>(t) * K + s];
      wsum += w[static_cast<long>(t) * K + s] * dw[static_cast<long>(t) * K + s];
    }
    for (int s = 0; s < K; ++s) {
      const float ws = w[static_cast<long>(t) * K + s];
      dl[s] = ws * (dw[static_cast<long>(t) * K + s] - wsum);
      if (lane == 0 && dlogit) dlogit[static_cast<long>(t) * K + s] = dl[s];
      if (lane == 0 && dl_perm) dl_perm[rows[s]] = dl[s];
    }
    if (coef8 && lane < 8) {  // dense dlogit row (E <= 8): the router weight-gradient coefficients
      float c = 0.f;
      for (int s = 0; s < K; ++s) c = (ex[s] == lane) ? dl[s] : c;
      coef8[static_cast<long>(t) * 8 + lane] = c;
    }
    // CU column segments per lane loaded before any is consumed (memory-level parallelism)
#ifndef HM_UNPERMUTE_CU
#define HM_UNPERMUTE_CU 2
#endif
    constexpr int CU = K <= 2 ? HM_UNPERMUTE_CU : 1;
    for (int q0 = lane; q0 < nv; q0 += 32 * CU) {
      uint4 v[CU][K], g[CU][K];
#pragma unroll
      for (int u = 0; u < CU; ++u)
        if (q0 + 32 * u < nv) {
#pragma unroll
          for (int s = 0; s < K; ++s) {
            v[u][s] = __ldg(reinterpret_cast<const uint4*>(dx_perm + static_cast<long>(rows[s]) * d) + q0 + 32 * u);
            g[u][s] = __ldg(reinterpret_cast<const uint4*>(wg_t + static_cast<long>(ex[s]) * d) + q0 + 32 * u);
          }
        }
#pragma unroll
      for (int u = 0; u < CU; ++u) {
        const int q = q0 + 32 * u;
        if (q >= nv) break;
        float acc[8];
#pragma unroll
        for (int z = 0; z < 8; ++z) acc[z] = 0.f;
#pragma unroll
        for (int s = 0; s < K; ++s) {
          const uint16_t* vh = reinterpret_cast<const uint16_t*>(&v[u][s]);
          const uint16_t* gh = reinterpret_cast<const uint16_t*>(&g[u][s]);
#pragma unroll
          for (int z = 0; z < 8; ++z) {
            acc[z] += bf16_to_f32(vh[z]);
            acc[z] = __fmaf_rn(dl[s], bf16_to_f32(gh[z]), acc[z]);
          }
        }
        uint4 o;
        o.x = pack_bf16x2(acc[0], acc[1]);
        o.y = pack_bf16x2(acc[2], acc[3]);
        o.z = pack_bf16x2(acc[4], acc[5]);
        o.w = pack_bf16x2(acc[6], acc[7]);
        reinterpret_cast<uint4*>(dx + static_cast<long>(t) * d)[q] = o;
      }
    }
  }
}

// v2 of the above, same arithmetic in the same order (bit-identical dx and dlogit): lanes s < K
// load token t's (row, expert, w, dw) once and broadcast them with shuffles (one round trip, not
// four dependent scalar-load chains per lane), the next token's are prefetched during this one's
// column loop, and (PF) the dx_perm rows of column group q + 32 are loaded while group q is
// summed. Measured (tools/router_bench.py): PF = false at 3 CTAs/SM is the fastest for k = 6
// (C3: 0.099 ms vs 0.109 with PF at 2 CTAs/SM and 0.121 for v1); v1 stays faster for k = 2.
template <int K, bool PF = true>
__global__ void __launch_bounds__(256, PF ? 2 : 3)
    unpermute_router_bwd2_kernel(const __nv_bfloat16* __restrict__ dx_perm,
                                 const int32_t* __restrict__ row_of, const int32_t* __restrict__ idx,
                                 const float* __restrict__ w, const float* __restrict__ dw,
                                 const __nv_bfloat16* __restrict__ wg_t, int T, int d,
                                 __nv_bfloat16* __restrict__ dx, float* __restrict__ dlogit,
                                 float* __restrict__ dl_perm, float* __restrict__ coef8 = nullptr) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int nv = d / 8;
  int mr = 0, me = 0;
  float mw = 0.f, md = 0.f;
  auto load_meta = [&](int tt) {
    if (tt < T && lane < K) {
      const long o = static_cast<long>(tt) * K + lane;
      mr = __ldg(row_of + o);
      me = __ldg(idx + o);
      mw = __ldg(w + o);
      md = __ldg(dw + o);
    }
  };
  load_meta(warp);
  for (int t = warp; t < T; t += nwarps) {
    int rows[K], ex[K];
    float ws[K], dws[K], dl[K];
#pragma unroll
    for (int s = 0; s < K; ++s) {
      rows[s] = __shfl_sync(0xffffffffu, mr, s);
      ex[s] = __shfl_sync(0xffffffffu, me, s);
      ws[s] = __shfl_sync(0xffffffffu, mw, s);
      dws[s] = __shfl_sync(0xffffffffu, md, s);
    }
    load_meta(t + nwarps);
    float wsum = 0.f;
#pragma unroll
    for (int s = 0; s < K; ++s) wsum = __fmaf_rn(ws[s], dws[s], wsum);
#pragma unroll
    for (int s = 0; s < K; ++s) {
      dl[s] = ws[s] * (dws[s] - wsum);
      if (lane == 0 && dlogit) dlogit[static_cast<long>(t) * K + s] = dl[s];
      if (lane == 0 && dl_perm) dl_perm[rows[s]] = dl[s];
    }
    if (coef8 && lane < 8) {  // dense dlogit row (E <= 8)
      float c = 0.f;
#pragma unroll
      for (int s = 0; s < K; ++s) c = (ex[s] == lane) ? dl[s] : c;
      coef8[static_cast<long>(t) * 8 + lane] = c;
    }
    uint4 cur[K];
#pragma unroll
    for (int s = 0; s < K; ++s)
      cur[s] = lane < nv ? __ldg(reinterpret_cast<const uint4*>(dx_perm + static_cast<long>(rows[s]) * d) + lane)
                         : make_uint4(0u, 0u, 0u, 0u);
    for (int q = lane; q < nv; q += 32) {
      uint4 nxt[K];
      const bool more = PF && q + 32 < nv;
#pragma unroll
      for (int s = 0; s < K; ++s)
        nxt[s] = more ? __ldg(reinterpret_cast<const uint4*>(dx_perm + static_cast<long>(rows[s]) * d) + q + 32)
                      : make_uint4(0u, 0u, 0u, 0u);
      float acc[8];
#pragma unroll
      for (int z = 0; z < 8; ++z) acc[z] = 0.f;
#pragma unroll
      for (int s = 0; s < K; ++s) {
        const uint4 g = __ldg(reinterpret_cast<const uint4*>(wg_t + static_cast<long>(ex[s]) * d) + q);
        const uint16_t* vh = reinterpret_cast<const uint16_t*>(&cur[s]);
        const uint16_t* gh = reinterpret_cast<const uint16_t*>(&g);
#pragma unroll
        for (int z = 0; z < 8; ++z) {
          acc[z] += bf16_to_f32(vh[z]);
          acc[z] = __fmaf_rn(dl[s], bf16_to_f32(gh[z]), acc[z]);
        }
      }
      uint4 o;
      o.x = pack_bf16x2(acc[0], acc[1]);
      o.y = pack_bf16x2(acc[2], acc[3]);
      o.z = pack_bf16x2(acc[4], acc[5]);
      o.w = pack_bf16x2(acc[6], acc[7]);
      reinterpret_cast<uint4*>(dx + static_cast<long>(t) * d)[q] = o;
      if (PF) {
#pragma unroll
        for (int s = 0; s < K; ++s) cur[s] = nxt[s];
      } else if (q + 32 < nv) {
#pragma unroll
        for (int s = 0; s < K; ++s)
          cur[s] = __ldg(reinterpret_cast<const uint4*>(dx_perm + static_cast<long>(rows[s]) * d) + q + 32);
      }
    }
  }
}

// plain unpermute-sum: dx[t] = sum_s dx_perm[row_of[t,s]]
template <int K>
__global__ void __launch_bounds__(256)
    unpermute_sum_kernel(const __nv_bfloat16* __restrict__ dx_perm, const int32_t* __restrict__ row_of,
                         int T, int d, __nv_bfloat16* __restrict__ dx) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int nv = d / 8;
  for (int t = warp; t < T; t += nwarps) {
    int rows[kMaxTopK];
    for (int s = 0; s < K; ++s) rows[s] = row_of[static_cast<long>(t) * K + s];
    for (int q = lane; q < nv; q += 32) {
      float acc[8];
#pragma unroll
      for (int z = 0; z < 8; ++z) acc[z] = 0.f;
      for (int s = 0; s < K; ++s) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(dx_perm + static_cast<long>(rows[s]) * d) + q);
        const uint16_t* vh = reinterpret_cast<const uint16_t*>(&v);
#pragma unroll
        for (int z = 0; z < 8; ++z) acc[z] += bf16_to_f32(vh[z]);
      }
      uint4 o;
      o.x = pack_bf16x2(acc[0], acc[1]);
      o.y = pack_bf16x2(acc[2], acc[3]);
      o.z = pack_bf16x2(acc[4], acc[5]);
      o.w = pack_bf16x2(acc[6], acc[7]);
      reinterpret_cast<uint4*>(dx + static_cast<long>(t) * d)[q] = o;
    }
  }
}

// ------------------------------------------------------------------------------------------
// Router weight gradient dWg[i,e] = sum over expert e's permuted rows r of dl_perm[r] * x_perm[r,i]
// (each token's routed copy carries its own dlogit). grid = (E * kWgSplit, ceil(d / 2048)); a
// thread owns 8 consecutive columns (one 16-byte load per row) and a slice of the expert's rows;
// per-split partial sums are reduced in split order by router_wgrad_reduce (deterministic).
constexpr int kWgSplit = 16;
__global__ void __launch_bounds__(256)
    router_wgrad_perm_kernel(const __nv_bfloat16* __restrict__ x_perm, const float* __restrict__ dl_perm,
                             const int32_t* __restrict__ offsets, int d, int E,
                             float* __restrict__ part /*[kWgSplit][E][d]*/) {
  const int e = blockIdx.x / kWgSplit;
  const int split = blockIdx.x % kWgSplit;
  const int col = (blockIdx.y * 256 + threadIdx.x) * 8;
  const int r0 = offsets[e], r1 = offsets[e + 1];
  const int n = r1 - r0;
  const int a = r0 + static_cast<int>((static_cast<long>(n) * split) / kWgSplit);
  const int b = r0 + static_cast<int>((static_cast<long>(n) * (split + 1)) / kWgSplit);
  float acc[8];
#pragma unroll
  for (int z = 0; z < 8; ++z) acc[z] = 0.f;
  if (col < d) {
    for (int r = a; r < b; ++r) {
      const float g = __ldg(dl_perm + r);
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(x_perm + static_cast<long>(r) * d + col));
      const uint16_t* h = reinterpret_cast<const uint16_t*>(&v);
#pragma unroll
      for (int z = 0; z < 8; ++z) acc[z] = __fmaf_rn(g, bf16_to_f32(h[z]), acc[z]);
    }
    float4* out = reinterpret_cast<float4*>(part + (static_cast<long>(split) * E + e) * d + col);
    out[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    out[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
}

// Token-major router weight gradient for E <= 8: dWg[i, e] = sum_t x[t, i] * dlogit_dense[t, e]
// (dlogit_dense = the selected experts' dlogits, zeros elsewhere — the dense formula autograd
// uses). Each token row is read ONCE (from its first routed copy, x_perm[row_of[t, 0]]) instead
// of once per routed copy: T*d*2 bytes instead of T*k*d*2. grid = (d / 64, kWgTokSplit); thread
// (tl, cg) = (tid / 8, tid % 8) owns columns [64*bx + 8*cg, +8) and tokens tl, tl + 32, ... of
// its split; a warp load covers 4 tokens x 128 contiguous bytes. Partials: fixed-order butterfly
// over the warp's 4 token lanes, then over the 8 warps in shared memory, then over the splits
// (router_wgrad_reduce) — deterministic.
constexpr int kWgTokSplit = 8;
constexpr int kWgTokUnroll = 4;
template <int K>
__global__ void __launch_bounds__(256, 2)
    router_wgrad_tok_kernel(const __nv_bfloat16* __restrict__ x_perm, const int32_t* __restrict__ row_of,
                            const int32_t* __restrict__ idx, const float* __restrict__ dlogit, int T,
                            int d, int E, float* __restrict__ part /*[kWgTokSplit][E][d]*/) {
  __shared__ float red[8][8][64];  // [warp][cg][e * 8 + z]
  const int tid = threadIdx.x;
  const int cg = tid & 7, tl = tid >> 3;
  const int warp = tid >> 5, lane = tid & 31;
  const int col = blockIdx.x * 64 + cg * 8;
  const int split = blockIdx.y;
  const int a = static_cast<int>((static_cast<long>(T) * split) / kWgTokSplit);
  const int b = static_cast<int>((static_cast<long>(T) * (split + 1)) / kWgTokSplit);
  constexpr int U = kWgTokUnroll;
  float acc[8][8];
#pragma unroll
  for (int e = 0; e < 8; ++e)
#pragma unroll
    for (int z = 0; z < 8; ++z) acc[e][z] = 0.f;
  // software pipeline: the row index and (expert, dlogit) pairs of group g+1 are loaded while
  // group g's rows are in flight, so each group costs one memory round trip, not two
  int row[U], ex[U][K];
  float dl[U][K];
  auto load_meta = [&](int t0) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = t0 + 32 * u;
      const bool ok = t < b;
      row[u] = ok ? __ldg(row_of + static_cast<long>(t) * K) : -1;
#pragma unroll
      for (int s = 0; s < K; ++s) {
        ex[u][s] = ok ? __ldg(idx + static_cast<long>(t) * K + s) : -1;
        dl[u][s] = ok ? __ldg(dlogit + static_cast<long>(t) * K + s) : 0.f;
      }
    }
  };
  load_meta(a + tl);
  for (int t0 = a + tl; t0 < b; t0 += 32 * U) {
    uint4 xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      xv[u] = row[u] >= 0 ? __ldg(reinterpret_cast<const uint4*>(x_perm + static_cast<long>(row[u]) * d + col))
                          : make_uint4(0u, 0u, 0u, 0u);
    int cex[U][K];
    float cdl[U][K];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int s = 0; s < K; ++s) { cex[u][s] = ex[u][s]; cdl[u][s] = dl[u][s]; }
    load_meta(t0 + 32 * U);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float coef[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float c = 0.f;
#pragma unroll
        for (int s = 0; s < K; ++s) c = (cex[u][s] == e) ? cdl[u][s] : c;
        coef[e] = c;
      }
      const uint16_t* h = reinterpret_cast<const uint16_t*>(&xv[u]);
#pragma unroll
      for (int z = 0; z < 8; z += 2) {
        const float2 xf = make_float2(bf16_to_f32(h[z]), bf16_to_f32(h[z + 1]));
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float2 r = __ffma2_rn(make_float2(coef[e], coef[e]), xf, make_float2(acc[e][z], acc[e][z + 1]));
          acc[e][z] = r.x;
          acc[e][z + 1] = r.y;
        }
      }
    }
  }
  // the warp's 4 token lanes (lane bits 3, 4) -> lanes 0..7
#pragma unroll
  for (int e = 0; e < 8; ++e)
#pragma unroll
    for (int z = 0; z < 8; ++z) {
      float v = acc[e][z];
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      acc[e][z] = v;
    }
  if (lane < 8) {
#pragma unroll
    for (int e = 0; e < 8; ++e)
#pragma unroll
      for (int z = 0; z < 8; ++z) red[warp][lane][e * 8 + z] = acc[e][z];
  }
  __syncthreads();
  // 8 cg x 64 (e, z) sums over the 8 warps; thread -> two of them
  for (int i = tid; i < 8 * 64; i += 256) {
    const int g = i >> 6, ez = i & 63;
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += red[w][g][ez];
    const int e = ez >> 3, z = ez & 7;
    const int c = blockIdx.x * 64 + g * 8 + z;
    if (e < E && c < d) part[(static_cast<long>(split) * E + e) * d + c] = s;
  }
}

// Router weight gradient for E <= 8 streamed through shared memory:
//   dWg[i, e] = sum_t x[t, i] * coef8[t, e]   (coef8 = the dense dlogit rows, zeros off the top-k)
// grid = (d / 512 column tiles, S token splits). Token rows [32 tokens x 512 columns] and their
// coefficient rows arrive by 1-D bulk copies (TMA engine; one row per lane of the producer warp
// 16) in a 4-stage ring. Compute warps 0..15: thread c = tid % 256 owns columns (2c, 2c+1) of the
// tile and 8 experts (16 fp32 accumulators, packed FFMA2 over the column pair); warps 0..7 take
// the even tokens of a stage, warps 8..15 the odd ones. Each thread sums in token order, the two
// halves are added (even + odd) at the end, and per-split partials are reduced in split order by
// router_wgrad_reduce_kernel: deterministic.
constexpr int kWgCols = 512;
constexpr int kWgTok = 32;
constexpr int kWgStages = 4;
constexpr int kWgXBytes = kWgTok * kWgCols * 2;   // 32 KB
constexpr int kWgCBytes = kWgTok * 8 * 4;          // 1 KB
constexpr int kWgStageBytes = kWgXBytes + kWgCBytes;
constexpr int kWgThreads = 17 * 32;
constexpr size_t router_wgrad_stream_smem_bytes() { return static_cast<size_t>(kWgStages) * kWgStageBytes + 128; }

__global__ void __launch_bounds__(kWgThreads, 1)
    router_wgrad_stream_kernel(const __nv_bfloat16* __restrict__ x, const float* __restrict__ coef8, int T,
                               int d, int E, float* __restrict__ part /*[S][E][d]*/) {
  extern __shared__ __align__(1024) uint8_t smem_wg[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_wg + kWgStages * kWgStageBytes);
  uint64_t* empty = full + kWgStages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c0 = blockIdx.x * kWgCols;
  const int S = gridDim.y, split = blockIdx.y;
  const int t_begin = static_cast<int>((static_cast<long>(T) * split) / S);
  const int t_end = static_cast<int>((static_cast<long>(T) * (split + 1)) / S);
  const int nst = (t_end - t_begin + kWgTok - 1) / kWgTok;
  if (tid == 0) {
    for (int s = 0; s < kWgStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 16);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == 16) {
    // ======== producer: lane r copies token row r of the stage, lane 0 arms the barrier ========
    for (int s = 0; s < nst; ++s) {
      const int slot = s % kWgStages;
      const int t0 = t_begin + s * kWgTok;
      const int nt = min(kWgTok, t_end - t0);
      if (s >= kWgStages) mbar_wait(&empty[slot], ((s / kWgStages) - 1) & 1);
      uint8_t* dst = smem_wg + slot * kWgStageBytes;
      if (lane == 0) {
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&full[slot], nt * kWgCols * 2 + nt * 32);
        bulk_load_1d(dst + kWgXBytes, coef8 + static_cast<long>(t0) * 8, nt * 32, &full[slot]);
      }
      __syncwarp();
      if (lane < nt)
        bulk_load_1d(dst + lane * kWgCols * 2, x + static_cast<long>(t0 + lane) * d + c0, kWgCols * 2, &full[slot]);
    }
    return;
  }
  const int c = tid & 255, par = tid >> 8;
  float2 acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = make_float2(0.f, 0.f);
  for (int s = 0; s < nst; ++s) {
    const int slot = s % kWgStages;
    const int nt = min(kWgTok, t_end - (t_begin + s * kWgTok));
    mbar_wait(&full[slot], (s / kWgStages) & 1);
    const uint8_t* st = smem_wg + slot * kWgStageBytes;
    const float* cf = reinterpret_cast<const float*>(st + kWgXBytes);
#pragma unroll 4
    for (int r = par; r < nt; r += 2) {
      const uint32_t xp = *reinterpret_cast<const uint32_t*>(st + r * kWgCols * 2 + c * 4);
      const float2 xf = make_float2(__uint_as_float(xp << 16), __uint_as_float(xp & 0xffff0000u));
      const float4 ca = *reinterpret_cast<const float4*>(cf + r * 8);
      const float4 cb = *reinterpret_cast<const float4*>(cf + r * 8 + 4);
      const float cc[8] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = __ffma2_rn(xf, make_float2(cc[e], cc[e]), acc[e]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  // even + odd token halves (fixed order), through the now idle ring (named barrier of the 16
  // compute warps: the producer warp has returned)
  asm volatile("bar.sync 1, 512;" ::: "memory");
  float2* xch = reinterpret_cast<float2*>(smem_wg);
  if (par == 1) {
#pragma unroll
    for (int e = 0; e < 8; ++e) xch[e * 256 + c] = acc[e];
  }
  asm volatile("bar.sync 1, 512;" ::: "memory");
  if (par == 0) {
    const int col = c0 + 2 * c;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float2 o = xch[e * 256 + c];
      const float2 v = make_float2(acc[e].x + o.x, acc[e].y + o.y);
      if (e < E && col < d) *reinterpret_cast<float2*>(part + (static_cast<long>(split) * E + e) * d + col) = v;
    }
  }
}

// ------------------------------------------------------------------------------------------
// Router backward in one streamed pass (E <= 8, k <= 3): per token row
//   dx[t]   = sum_s dx_perm[row_of[t,s]] + dlogit[t,s] * Wg[:, idx[t,s]]   (the unpermute kernel's
//             per-element order: acc += dx_perm; acc = fma(dlogit, wg, acc), slot by slot)
//   dWg    += x[t] (x) dlogit_dense[t]
// so x and the routed dX rows are each read once, dx is written once, and the dWg FMAs run under
// the HBM stream instead of in a second pass. router_dlogit_kernel first writes a 64-byte record
// per token: [0..8) dense dlogit row, [8..8+k) dlogit by slot, [12..12+k) expert by slot.
constexpr int kRbCols = 1024;  // columns per CTA tile (512 compute threads x 2 columns)
constexpr int kRbTok = 8;      // tokens per stage (8 x (1 + k) bulk copies of 2 KB)
constexpr int kRbMeta = 16;    // floats per token record

template <int K>
__global__ void router_dlogit_kernel(const int32_t* __restrict__ idx, const float* __restrict__ w,
                                     const float* __restrict__ dw, int T, float* __restrict__ meta,
                                     float* __restrict__ dlogit) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  float ws[K], dws[K];
  int ex[K];
  float wsum = 0.f;
#pragma unroll
  for (int s = 0; s < K; ++s) {
    ws[s] = w[static_cast<long>(t) * K + s];
    dws[s] = dw[static_cast<long>(t) * K + s];
    ex[s] = idx[static_cast<long>(t) * K + s];
    wsum = __fmaf_rn(ws[s], dws[s], wsum);
  }
  float rec[kRbMeta];
#pragma unroll
  for (int q = 0; q < kRbMeta; ++q) rec[q] = 0.f;
#pragma unroll
  for (int s = 0; s < K; ++s) {
    const float dl = ws[s] * (dws[s] - wsum);
    if (dlogit) dlogit[static_cast<long>(t) * K + s] = dl;
#pragma unroll
    for (int e = 0; e < 8; ++e) rec[e] = (ex[s] == e) ? dl : rec[e];
    rec[8 + s] = dl;
    rec[12 + s] = __int_as_float(ex[s]);
  }
  float4* o = reinterpret_cast<float4*>(meta + static_cast<long>(t) * kRbMeta);
#pragma unroll
  for (int q = 0; q < 4; ++q) o[q] = make_float4(rec[4 * q], rec[4 * q + 1], rec[4 * q + 2], rec[4 * q + 3]);
}

template <int K>
struct RbCfg {
  static constexpr int kStages = K <= 2 ? 4 : 3;
  static constexpr int kXBytes = kRbTok * kRbCols * 2;        // 16 KB
  static constexpr int kDBytes = kRbTok * K * kRbCols * 2;    // 16 KB per slot
  static constexpr int kMBytes = kRbTok * kRbMeta * 4;         // 512 B
  static constexpr int kStageBytes = kXBytes + kDBytes + kMBytes;
  static constexpr int kWgBytes = 8 * kRbCols * 2;             // Wg^T tile, bf16
  static constexpr size_t kSmem = static_cast<size_t>(kStages) * kStageBytes + kWgBytes + 128;
};

template <int K>
__global__ void __launch_bounds__(17 * 32, 1)
    router_bwd_fused_kernel(const __nv_bfloat16* __restrict__ dx_perm, const int32_t* __restrict__ row_of,
                            const float* __restrict__ meta, const __nv_bfloat16* __restrict__ x,
                            const __nv_bfloat16* __restrict__ wg_t, int T, int d, int E,
                            __nv_bfloat16* __restrict__ dx, float* __restrict__ part /*[S][E][d]*/) {
  using C = RbCfg<K>;
  extern __shared__ __align__(1024) uint8_t smem_rb[];
  uint32_t* wgs = reinterpret_cast<uint32_t*>(smem_rb + C::kStages * C::kStageBytes);  // [8][512] bf16 pairs
  uint64_t* full = reinterpret_cast<uint64_t*>(wgs + 8 * (kRbCols / 2));
  uint64_t* empty = full + C::kStages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c0 = blockIdx.x * kRbCols;
  const int S = gridDim.y, split = blockIdx.y;
  const int t_begin = static_cast<int>((static_cast<long>(T) * split) / S);
  const int t_end = static_cast<int>((static_cast<long>(T) * (split + 1)) / S);
  const int nst = (t_end - t_begin + kRbTok - 1) / kRbTok;
  if (tid == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 16);
    }
    fence_barrier_init();
  }
  if (tid < 16 * 32) {  // the Wg^T tile (bf16 pairs; zeros past E)
    for (int i = tid; i < 8 * (kRbCols / 2); i += 16 * 32) {
      const int e = i / (kRbCols / 2), c = i % (kRbCols / 2);
      wgs[i] = (e < E) ? *reinterpret_cast<const uint32_t*>(wg_t + static_cast<long>(e) * d + c0 + 2 * c) : 0u;
    }
  }
  __syncthreads();
  if (warp == 16) {
    // ======== producer: lane r * (1 + K) + q copies token r's x tile (q = 0) / routed dX tile q ========
    for (int s = 0; s < nst; ++s) {
      const int slot = s % C::kStages;
      const int t0 = t_begin + s * kRbTok;
      const int nt = min(kRbTok, t_end - t0);
      if (s >= C::kStages) mbar_wait(&empty[slot], ((s / C::kStages) - 1) & 1);
      uint8_t* st = smem_rb + slot * C::kStageBytes;
      if (lane == 0) {
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&full[slot], nt * (1 + K) * kRbCols * 2 + nt * kRbMeta * 4);
        bulk_load_1d(st + C::kXBytes + C::kDBytes, meta + static_cast<long>(t0) * kRbMeta, nt * kRbMeta * 4, &full[slot]);
      }
      __syncwarp();
      const int r = lane / (1 + K), q = lane % (1 + K);
      if (r < nt && lane < kRbTok * (1 + K)) {
        const long t = t0 + r;
        if (q == 0) {
          bulk_load_1d(st + r * kRbCols * 2, x + t * d + c0, kRbCols * 2, &full[slot]);
        } else {
          const long row = __ldg(row_of + t * K + (q - 1));
          bulk_load_1d(st + C::kXBytes + (r * K + (q - 1)) * kRbCols * 2, dx_perm + row * d + c0, kRbCols * 2,
                       &full[slot]);
        }
      }
    }
  } else {
    // ======== compute: thread c owns columns (2c, 2c + 1) of the tile, every token ========
    const int c = tid;
    float2 acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = make_float2(0.f, 0.f);
    for (int s = 0; s < nst; ++s) {
      const int slot = s % C::kStages;
      const int t0 = t_begin + s * kRbTok;
      const int nt = min(kRbTok, t_end - t0);
      mbar_wait(&full[slot], (s / C::kStages) & 1);
      const uint8_t* st = smem_rb + slot * C::kStageBytes;
      const float* mt = reinterpret_cast<const float*>(st + C::kXBytes + C::kDBytes);
#pragma unroll 2
      for (int r = 0; r < nt; ++r) {
        const float* rec = mt + r * kRbMeta;
        const float4 ca = *reinterpret_cast<const float4*>(rec);
        const float4 cb = *reinterpret_cast<const float4*>(rec + 4);
        const float4 dls = *reinterpret_cast<const float4*>(rec + 8);
        const float4 exs = *reinterpret_cast<const float4*>(rec + 12);
        const float dl[4] = {dls.x, dls.y, dls.z, dls.w};
        const int ex[4] = {__float_as_int(exs.x), __float_as_int(exs.y), __float_as_int(exs.z), __float_as_int(exs.w)};
        float2 o = make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < K; ++q) {
          const uint32_t v = *reinterpret_cast<const uint32_t*>(st + C::kXBytes + (r * K + q) * kRbCols * 2 + c * 4);
          const uint32_t gp = wgs[ex[q] * (kRbCols / 2) + c];
          o.x += __uint_as_float(v << 16);
          o.y += __uint_as_float(v & 0xffff0000u);
          o.x = __fmaf_rn(dl[q], __uint_as_float(gp << 16), o.x);
          o.y = __fmaf_rn(dl[q], __uint_as_float(gp & 0xffff0000u), o.y);
        }
        *reinterpret_cast<uint32_t*>(dx + static_cast<long>(t0 + r) * d + c0 + 2 * c) = pack_bf16x2(o.x, o.y);
        const uint32_t xp = *reinterpret_cast<const uint32_t*>(st + r * kRbCols * 2 + c * 4);
        const float2 xf = make_float2(__uint_as_float(xp << 16), __uint_as_float(xp & 0xffff0000u));
        const float cc[8] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = __ffma2_rn(xf, make_float2(cc[e], cc[e]), acc[e]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
    const int col = c0 + 2 * c;
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (e < E) *reinterpret_cast<float2*>(part + (static_cast<long>(split) * E + e) * d + col) = acc[e];
  }
}

// Dense bf16 dlogit rows dl[T][E] (zero except the k routed experts of each token) from the
// per-slot dlogits in token order, and the K-split segment table {0, T/S, ..., T}: the operands
// of the router weight gradient as one tensor-core GEMM, dWg^T[E][d] = sum_t dl[t]^T x[t]
// (E > 8: each token row of x read once, instead of once per routed copy).
template <int K>
__global__ void __launch_bounds__(256)
    dense_dlogit_kernel(const int32_t* __restrict__ idx, const float* __restrict__ dl_tok, int T, int E,
                        int S, __nv_bfloat16* __restrict__ dl, int32_t* __restrict__ seg) {
  if (blockIdx.x == 0 && threadIdx.x <= S) seg[threadIdx.x] = static_cast<int>(static_cast<long>(T) * threadIdx.x / S);
  const int nc = E >> 3;
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<long>(T) * nc) return;
  const int t = static_cast<int>(i / nc), c = static_cast<int>(i % nc);
  float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int s = 0; s < K; ++s) {
    const int e = idx[static_cast<long>(t) * K + s];
    if ((e >> 3) == c) v[e & 7] = dl_tok[static_cast<long>(t) * K + s];
  }
  *reinterpret_cast<uint4*>(dl + static_cast<long>(t) * E + c * 8) =
      make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
}

__global__ void router_wgrad_reduce_kernel(const float* __restrict__ part, int nsplit, int d, int E,
                                           __nv_bfloat16* __restrict__ dwg /*[d][E]*/) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<long>(d) * E) return;
  const int col = static_cast<int>(i / E), e = static_cast<int>(i % E);
  float s = 0.f;
  for (int p = 0; p < nsplit; ++p) s += part[(static_cast<long>(p) * E + e) * d + col];
  dwg[i] = __float2bfloat16_rn(s);
}


// ------------------------------------------------------------------------------------------
// NVLink peer-memory transport (the fused dispatch / combine of the ZP executor).
//
// Fused permute + dispatch: each token row is read once and written (a) optionally to the local
// permuted buffer and (b) straight into the receive buffer of the expert's owner, which may be
// another GPU (a peer-mapped pointer): row (t, s) of expert e lands at
//   dest_base[e] + (dest_start[e] + (row_of[t,s] - offsets[e])) * d.
template <int VPL>
__global__ void __launch_bounds__(256)
    dispatch_permute_p2p_kernel(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ idx,
                                const int32_t* __restrict__ chunk_base, const int32_t* __restrict__ offsets,
                                int T, int d, int E, int k, __nv_bfloat16* __restrict__ x_perm,
                                int32_t* __restrict__ row_src, int32_t* __restrict__ row_of,
                                const unsigned long long* __restrict__ dest_base,
                                const int32_t* __restrict__ dest_start) {
  __shared__ int s_idx[kChunk * kMaxTopK];
  __shared__ int s_row[kChunk * kMaxTopK];
  const int c = blockIdx.x;
  const int tbeg = c * kChunk;
  const int nt = min(kChunk, T - tbeg);
  for (int i = threadIdx.x; i < nt * k; i += blockDim.x) s_idx[i] = idx[static_cast<long>(tbeg) * k + i];
  __syncthreads();
  assign_rows_ballot(s_idx, s_row, chunk_base + static_cast<long>(c) * E, nt * k, E);
  __syncthreads();
  if (blockIdx.y == 0) {
    for (int i = threadIdx.x; i < nt * k; i += blockDim.x) {
      const int r = s_row[i];
      row_of[static_cast<long>(tbeg) * k + i] = r;
      if (row_src) row_src[r] = tbeg + i / k;
    }
  }
  // gridDim.y CTAs per chunk, as in dispatch_permute_kernel
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (VPL == 0) {  // any d % 8 == 0: the row in pieces of 8 x 32 16-byte vectors
    const int nv = d / 8;
    for (int tt = warp + 8 * blockIdx.y; tt < nt; tt += 8 * gridDim.y) {
      const long t = tbeg + tt;
      const uint4* src = reinterpret_cast<const uint4*>(x + t * d);
      for (int q0 = 0; q0 < nv; q0 += 256) {
        uint4 v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (q0 + 32 * i + lane < nv) v[i] = __ldg(src + q0 + 32 * i + lane);
        for (int s = 0; s < k; ++s) {
          const int r = s_row[tt * k + s];
          const int e = s_idx[tt * k + s];
          uint4* dl = x_perm ? reinterpret_cast<uint4*>(x_perm + static_cast<long>(r) * d) : nullptr;
          uint4* dp = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(dest_base[e]) +
                                               (static_cast<long>(dest_start[e]) + r - offsets[e]) * d);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int q = q0 + 32 * i + lane;
            if (q < nv) {
              if (dl) dl[q] = v[i];
              dp[q] = v[i];
            }
          }
        }
      }
    }
    return;
  }
  for (int tt = warp + 8 * blockIdx.y; tt < nt; tt += 8 * gridDim.y) {
    const long t = tbeg + tt;
    const uint4* src = reinterpret_cast<const uint4*>(x + t * d);
    uint4 v[VPL > 0 ? VPL : 1];
#pragma unroll
    for (int q = 0; q < VPL; ++q) v[q] = __ldg(src + q * 32 + lane);
    for (int s = 0; s < k; ++s) {
      const int r = s_row[tt * k + s];
      const int e = s_idx[tt * k + s];
      if (x_perm) {
        uint4* dst = reinterpret_cast<uint4*>(x_perm + static_cast<long>(r) * d);
#pragma unroll
        for (int q = 0; q < VPL; ++q) dst[q * 32 + lane] = v[q];
      }
      __nv_bfloat16* peer = reinterpret_cast<__nv_bfloat16*>(dest_base[e]) +
                            (static_cast<long>(dest_start[e]) + r - offsets[e]) * d;
      uint4* dst = reinterpret_cast<uint4*>(peer);
#pragma unroll
      for (int q = 0; q < VPL; ++q) dst[q * 32 + lane] = v[q];
    }
  }
}

// Fused combine backward + dispatch of dY: dy_perm row (t, s) = w[t,s] * dy[t] goes straight to
// the owner's receive buffer (same addressing as the forward dispatch); dw[t,s] = <dy[t], y_perm[row]>.
template <int K>
__global__ void __launch_bounds__(256)
    combine_bwd_p2p_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ y_perm,
                           const int32_t* __restrict__ row_of, const int32_t* __restrict__ idx,
                           const float* __restrict__ w, const int32_t* __restrict__ offsets, int T, int d,
                           const unsigned long long* __restrict__ dest_base,
                           const int32_t* __restrict__ dest_start, float* __restrict__ dw) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int nv = d / 8;
  for (int t = warp; t < T; t += nwarps) {
    int rows[K];
    float ws[K], dot[K];
    uint4* dsts[K];
    for (int s = 0; s < K; ++s) {
      rows[s] = row_of[static_cast<long>(t) * K + s];
      ws[s] = w[static_cast<long>(t) * K + s];
      dot[s] = 0.f;
      const int e = idx[static_cast<long>(t) * K + s];
      dsts[s] = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(dest_base[e]) +
                                         (static_cast<long>(dest_start[e]) + rows[s] - offsets[e]) * d);
    }
    for (int q = lane; q < nv; q += 32) {
      const uint4 g = __ldg(reinterpret_cast<const uint4*>(dy + static_cast<long>(t) * d) + q);
      const uint16_t* gh = reinterpret_cast<const uint16_t*>(&g);
      float gf[8];
#pragma unroll
      for (int z = 0; z < 8; ++z) gf[z] = bf16_to_f32(gh[z]);
      for (int s = 0; s < K; ++s) {
        const uint4 yv = __ldg(reinterpret_cast<const uint4*>(y_perm + static_cast<long>(rows[s]) * d) + q);
        const uint16_t* yh = reinterpret_cast<const uint16_t*>(&yv);
#pragma unroll
        for (int z = 0; z < 8; ++z) dot[s] = __fmaf_rn(gf[z], bf16_to_f32(yh[z]), dot[s]);
        uint4 o;
        o.x = pack_bf16x2(ws[s] * gf[0], ws[s] * gf[1]);
        o.y = pack_bf16x2(ws[s] * gf[2], ws[s] * gf[3]);
        o.z = pack_bf16x2(ws[s] * gf[4], ws[s] * gf[5]);
        o.w = pack_bf16x2(ws[s] * gf[6], ws[s] * gf[7]);
        dsts[s][q] = o;
      }
    }
    for (int s = 0; s < K; ++s) {
      float v = dot[s];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) dw[static_cast<long>(t) * K + s] = v;
    }
  }
}

// Completion signalling between GPUs: after the data writes of this stream completed, add 1 to
// each listed (peer-mapped) 32-bit counter with release semantics at system scope.
constexpr int kMaxPeers = 8;
// ------------------------------------------------------------------------------------------
// Device-side receive layout of one (layer, micro-batch) exchange (ZP peer-memory transport).
// Every CTA rebuilds the small tables (<= kZpMaxSenders x 256 counts) in shared memory; CTA 0
// writes the sender table, the owner's segments, pool bases and GEMM row shifts; all CTAs fill
// the per-row return addresses of the owner's received rows (grid-stride over the rows).
// Receive slot of owner o: its experts in id order, inside an expert the senders in rank order.
constexpr int kZpMaxSenders = 8;
constexpr int kZpMaxPeersLayout = 16;  // ranks of the exchange (owners)
constexpr int kZpLayoutThreads = 256;
constexpr int kZpLayoutRowsPerCta = 2048;

__global__ void __launch_bounds__(kZpLayoutThreads)
    zp_layout_kernel(const int32_t* __restrict__ counts_all, int M, int E, const int32_t* __restrict__ owners,
                     int me, int n_own, int cap, const unsigned long long* __restrict__ y_base,
                     long long dx_delta, int row_bytes, int32_t* __restrict__ dest_start,
                     int32_t* __restrict__ seg, unsigned long long* __restrict__ out_rows_y,
                     unsigned long long* __restrict__ out_rows_dx, int32_t* __restrict__ shifts,
                     int32_t* __restrict__ top, int pool_base, int pool_rows, int32_t* __restrict__ err) {
  __shared__ int s_cnt[kZpMaxSenders][256];
  __shared__ int s_off[kZpMaxSenders][256];  // sender a's first permuted row of expert e
  __shared__ int s_start[256];               // first row of expert e in its owner's slot
  __shared__ int s_own[256];
  __shared__ int s_seg_row[kZpMaxSenders * 256 + 1];  // my received segments (expert-major, sender-minor)
  __shared__ int s_seg_src[kZpMaxSenders * 256];      // ... their sender rank
  __shared__ int s_seg_off[kZpMaxSenders * 256];      // ... their first row in the sender's permuted buffer
  __shared__ int s_nseg, s_total;
  const int tid = threadIdx.x;
  for (int i = tid; i < M * E; i += blockDim.x) s_cnt[i / E][i % E] = counts_all[i];
  for (int e = tid; e < E; e += blockDim.x) s_own[e] = owners[e];
  __syncthreads();
  if (tid < M) {  // sender offsets: exclusive prefix over the experts
    int a = 0;
    for (int e = 0; e < E; ++e) {
      s_off[tid][e] = a;
      a += s_cnt[tid][e];
    }
  }
  if (tid == kZpLayoutThreads - 1) {  // owners' slots: experts in id order
    int run[kZpMaxPeersLayout];
    for (int o = 0; o < kZpMaxPeersLayout; ++o) run[o] = 0;
    for (int e = 0; e < E; ++e) {
      int tot = 0;
      for (int a = 0; a < M; ++a) tot += s_cnt[a][e];
      const int o = s_own[e];
      if (o < 0 || o >= kZpMaxPeersLayout) {  // not a rank of the exchange: flag, place nowhere
        atomicOr(err, 8);
        s_start[e] = 0;
        continue;
      }
      s_start[e] = run[o];
      run[o] += tot;
    }
    s_total = run[me];
  }
  __syncthreads();
  if (tid == 0) {  // my received segments, in slot order
    int n = 0;
    for (int e = 0; e < E; ++e) {
      if (s_own[e] != me) continue;
      int r = s_start[e];
      for (int a = 0; a < M; ++a) {
        s_seg_row[n] = r;
        s_seg_src[n] = a;
        s_seg_off[n] = s_off[a][e];
        r += s_cnt[a][e];
        ++n;
      }
    }
    s_seg_row[n] = s_total;
    s_nseg = n;
  }
  __syncthreads();
  const int total = s_total;
  if (blockIdx.x == 0) {
    if (me < M)
      for (int e = tid; e < E; e += blockDim.x) {
        int st = s_start[e];
        for (int a = 0; a < me; ++a) st += s_cnt[a][e];
        dest_start[e] = st;
      }
    if (tid == 0 && n_own > 0) {
      // bump-allocate this micro-batch's rows in the layer's pool region
      int bad = total > cap ? 4 : 0;
      const int used = *top;
      if (used + total > pool_rows) bad |= 1;
      if (!bad) *top = used + total;
      else atomicOr(err, bad);
      int i = 0;
      for (int e = 0; e < E && i < n_own; ++e)
        if (s_own[e] == me) seg[i++] = bad ? 0 : s_start[e];
      for (; i <= n_own; ++i) seg[i] = bad ? 0 : total;
      const int f = pool_base + (bad ? 0 : used);
      // {a, o} row shifts: up+gate {0, f}, down {f, 0}, SwiGLU backward {0, f}, dX {f, 0}
      shifts[0] = 0; shifts[1] = f; shifts[2] = f; shifts[3] = 0;
      shifts[4] = 0; shifts[5] = f; shifts[6] = f; shifts[7] = 0;
    }
  }
  if (n_own <= 0) return;
  const int nseg = s_nseg;
  const int rmax = total < cap ? total : cap;
  for (int r = blockIdx.x * blockDim.x + tid; r < rmax; r += gridDim.x * blockDim.x) {
    int lo = 0, hi = nseg - 1;  // last segment whose first row <= r (empty segments share rows)
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_seg_row[mid] <= r) lo = mid;
      else hi = mid - 1;
    }
    const long row = s_seg_off[lo] + (r - s_seg_row[lo]);
    const unsigned long long ya = y_base[s_seg_src[lo]] + static_cast<unsigned long long>(row) * row_bytes;
    out_rows_y[r] = ya;
    out_rows_dx[r] = ya + dx_delta;
  }
}

struct PeerFlags {
  unsigned long long ptr[kMaxPeers];
};
struct FlagTargets {
  unsigned int v[kMaxPeers];
};

__global__ void signal_add_kernel(const __grid_constant__ PeerFlags flags, int n) {
  const int i = threadIdx.x;
  if (i < n) {
    __threadfence_system();
    unsigned int* f = reinterpret_cast<unsigned int*>(flags.ptr[i]);
    asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(f) : "memory");
  }
}

// Wait (acquire, system scope) until local counters flags[i*stride] reach targets[i]. The
// counters are written by peers over NVLink, never by another kernel of this GPU.
__global__ void wait_geq_kernel(const unsigned int* __restrict__ flags, int stride,
                                const __grid_constant__ FlagTargets targets, int n) {
  const int i = threadIdx.x;
  if (i < n) {
    const unsigned int want = targets.v[i];
    const unsigned int* f = flags + static_cast<long>(i) * stride;
    unsigned int v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    } while (static_cast<int>(v - want) < 0);
  }
}

// bf16 transpose [R][C] -> [C][R] (router weight layout helper)
__global__ void transpose_bf16_kernel(const __nv_bfloat16* __restrict__ in, int R, int C,
                                      __nv_bfloat16* __restrict__ out) {
  __shared__ __nv_bfloat16 tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int r = by + j, c = bx + threadIdx.x;
    if (r < R && c < C) tile[j][threadIdx.x] = in[static_cast<long>(r) * C + c];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int c = bx + j, r = by + threadIdx.x;
    if (r < R && c < C) out[static_cast<long>(c) * R + r] = tile[threadIdx.x][j];
  }
}

}  // namespace hm
