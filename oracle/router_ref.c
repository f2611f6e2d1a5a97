/* router_ref.c — C restatement of the router/dispatch semantics (TEST INFRASTRUCTURE ONLY).
 *
 * Same contract as oracle/moe_oracle.py (router_logits / topk_softmax / permutation), written
 * in plain C so the bit-exact routing check also runs at the full C2/C3 sizes in seconds.
 * Parity status: "parity unpinned" — the reference has no router code; the
 * semantics follow PAPER.md:110,358 and the fixed summation order documented in
 * paper_2504_03871_b200/csrc/moe_kernels.cuh.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline float bf16(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* logits[t,e], blocked order: for each 256-wide block j, lane L accumulates i = 256*j + 8*L + q
 * (q = 0..7) from 0 with one rounding per step (bf16 products are exact in fp32), an xor
 * butterfly 16, 8, 4, 2, 1 combines the 32 lanes into the block partial P_j, and the logit is
 * ((P_0 + P_1) + P_2) + ... in block order. */
void hm_ref_router_logits(const uint16_t* x, const uint16_t* wg, int T, int d, int E, float* out) {
  const int nj = d / 256;
#pragma omp parallel for schedule(static)
  for (int t = 0; t < T; ++t) {
    float lane[32];
    for (int e = 0; e < E; ++e) {
      float total = 0.0f;
      for (int j = 0; j < nj; ++j) {
        for (int L = 0; L < 32; ++L) {
          float acc = 0.0f;
          for (int q = 0; q < 8; ++q) {
            const int i = 256 * j + 8 * L + q;
            volatile float prod = bf16(x[(long)t * d + i]) * bf16(wg[(long)i * E + e]);
            acc = acc + prod;
          }
          lane[L] = acc;
        }
        for (int off = 16; off > 0; off >>= 1) {
          float nxt[32];
          for (int L = 0; L < 32; ++L) nxt[L] = lane[L] + lane[L ^ off];
          memcpy(lane, nxt, sizeof(lane));
        }
        total = (j == 0) ? lane[0] : total + lane[0];
      }
      out[(long)t * E + e] = total;
    }
  }
}

/* ranking of the top-k: larger logit first, ties -> lower expert id, NaN after every number
 * (including -inf), NaN ties -> lower id; a selected expert is never selected again. This is the
 * total order (isnan, -logit, id) that numpy's lexsort in moe_oracle.topk_softmax also applies. */
static int ranks_before(float a, int ea, float b, int eb) {
  const int na = isnan(a), nb = isnan(b);
  if (na != nb) return nb;           /* a number ranks before NaN */
  if (!na && a != b) return a > b;   /* both numbers: larger first */
  return ea < eb;                    /* equal numbers, or both NaN: lower id first */
}

/* top-k and softmax over the selected logits */
void hm_ref_topk_softmax(const float* logits, int T, int E, int k, int32_t* idx, float* w) {
#pragma omp parallel for schedule(static)
  for (int t = 0; t < T; ++t) {
    const float* l = logits + (long)t * E;
    int sel[8];
    for (int s = 0; s < k; ++s) {
      int best = -1;
      for (int e = 0; e < E; ++e) {
        int used = 0;
        for (int p = 0; p < s; ++p) used |= (sel[p] == e);
        if (used) continue;
        if (best < 0 || ranks_before(l[e], e, l[best], best)) best = e;
      }
      sel[s] = best;
    }
    float ex[8], sum = 0.0f;
    for (int s = 0; s < k; ++s) {
      ex[s] = expf(l[sel[s]] - l[sel[0]]);
      sum += ex[s];
    }
    for (int s = 0; s < k; ++s) {
      idx[(long)t * k + s] = sel[s];
      w[(long)t * k + s] = ex[s] / sum;
    }
  }
}

/* stable (expert, token) permutation: counts, offsets, row_src[T*k], row_of[T*k] */
void hm_ref_permutation(const int32_t* idx, int T, int k, int E, int32_t* counts, int32_t* offsets,
                        int32_t* row_src, int32_t* row_of) {
  memset(counts, 0, sizeof(int32_t) * E);
  for (long i = 0; i < (long)T * k; ++i) counts[idx[i]]++;
  offsets[0] = 0;
  for (int e = 0; e < E; ++e) offsets[e + 1] = offsets[e] + counts[e];
  int32_t* next = (int32_t*)malloc(sizeof(int32_t) * E);
  memcpy(next, offsets, sizeof(int32_t) * E);
  for (int t = 0; t < T; ++t)
    for (int s = 0; s < k; ++s) {
      const int e = idx[(long)t * k + s];
      const int r = next[e]++;
      row_src[r] = t;
      row_of[(long)t * k + s] = r;
    }
  free(next);
}
