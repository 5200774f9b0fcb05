// K3: busiest expert-parallel shard under power-law expert popularity, one
// warp per (pooled tokens, ep) -- restates moe_load.tokens_per_expert +
// expert_shard_tokens + busiest_shard_tokens (moe_load.py:67-147) exactly:
//   raw_i = fl(q_i * target), q_i = fl(w_i / sum(w)) from numpy on the host,
//   counts = floor(raw); the `short` largest fractional parts (ties -> lower
//   expert index, i.e. np.lexsort((arange, -frac))) get +1; counts above the
//   per-expert ceiling spill in by-weight order; result = max over contiguous
//   EP blocks of the block sums.
// The top-`short` selection is an exact warp radix-select over the IEEE bit
// patterns of the fractions (monotone for non-negative doubles): 8-bit digits
// starting at the highest bit where the fractions differ, a 256-bin shared
// histogram per level, and index order for fully tied keys.
#pragma once
#include <stdint.h>
#include <math.h>

namespace lc {

__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ uint64_t warp_or_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ uint64_t warp_and_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v &= __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// exclusive prefix over lanes (lane order) of a small int
__device__ __forceinline__ int warp_excl_scan(int v, int lane) {
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x - v;
}

// hist: 256 ints of shared memory private to this warp.
// Per-lane expert counts (experts lane*per .. lane*per+per-1) of
// tokens_per_expert: they depend on (q, total, topk) only, not on ep.
template <int PER>
__device__ __forceinline__ void warp_expert_counts(const double* __restrict__ q, const double* __restrict__ order,
                                                   int E, int64_t total, int64_t topk, int* hist, int64_t (&cnt)[PER]) {
  const int lane = threadIdx.x & 31;
  const int per = (E + 31) >> 5;  // experts per lane, contiguous
  uint64_t key[PER];
  const int64_t target = total * topk;
  const double tgt = (double)target;
  int64_t local = 0;
  uint64_t kor = 0, kand = ~0ull;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int i = lane * per + j;
    cnt[j] = 0;
    key[j] = 0;
    if (j < per && i < E) {
      const double raw = q[i] * tgt;
      cnt[j] = (int64_t)floor(raw);
      const double fr = raw - (double)cnt[j];
      key[j] = (uint64_t)__double_as_longlong(fr);
      local += cnt[j];
      kor |= key[j];
      kand &= key[j];
    }
  }
  const int64_t shortfall = target - warp_sum_i64(local);
  uint32_t sel = 0;  // bit j: element j gets +1
  if (shortfall > 0) {
    uint32_t cand = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j)
      if (j < per && lane * per + j < E) cand |= 1u << j;
    int64_t need = shortfall;
    const uint64_t diff = warp_or_u64(kor) ^ warp_and_u64(kand);
    int shift = diff ? (63 - __clzll((long long)diff)) - 7 : -8;
    if (shift < 0 && diff) shift = 0;
    while (true) {
      if (shift < 0) {
        // remaining candidates have identical keys: lowest indices first
        int c = __popc(cand);
        const int before = warp_excl_scan(c, lane);
#pragma unroll
        for (int j = 0; j < PER; ++j)
          if (cand & (1u << j)) {
            if (before + __popc(cand & ((1u << j) - 1)) < need) sel |= 1u << j;
          }
        break;
      }
#pragma unroll
      for (int b = 0; b < 8; ++b) hist[lane * 8 + b] = 0;
      __syncwarp();
#pragma unroll
      for (int j = 0; j < PER; ++j)
        if (cand & (1u << j)) atomicAdd(&hist[(int)((key[j] >> shift) & 0xff)], 1);
      __syncwarp();
      int h[8];
      int lane_tot = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) { h[b] = hist[lane * 8 + b]; lane_tot += h[b]; }
      __syncwarp();
      // suffix sum over higher lanes (higher digits)
      int suf = lane_tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_down_sync(0xffffffffu, suf, o);
        if (lane + o < 32) suf += y;
      }
      int64_t above = (int64_t)(suf - lane_tot);  // candidates in digits owned by higher lanes
      int found_digit = -1;
      int64_t found_above = 0;
      int found_cnt = 0;
#pragma unroll
      for (int b = 7; b >= 0; --b) {
        if (found_digit < 0 && above < need && above + h[b] >= need) {
          found_digit = lane * 8 + b;
          found_above = above;
          found_cnt = h[b];
        }
        above += h[b];
      }
      const unsigned who = __ballot_sync(0xffffffffu, found_digit >= 0);
      const int src = __ffs(who) - 1;
      const int D = __shfl_sync(0xffffffffu, found_digit, src);
      const int64_t cnt_above = __shfl_sync(0xffffffffu, found_above, src);
      const int inD = __shfl_sync(0xffffffffu, found_cnt, src);
#pragma unroll
      for (int j = 0; j < PER; ++j)
        if (cand & (1u << j)) {
          const int dg = (int)((key[j] >> shift) & 0xff);
          if (dg > D) { sel |= 1u << j; cand &= ~(1u << j); }
          else if (dg < D) cand &= ~(1u << j);
        }
      need -= cnt_above;
      if (need == inD) {  // every remaining candidate is selected
        sel |= cand;
        break;
      }
      shift = shift == 0 ? -1 : (shift >= 8 ? shift - 8 : 0);
    }
  }
  bool over = false;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    cnt[j] += (sel >> j) & 1u;
    over |= cnt[j] > total;
  }
  if (__any_sync(0xffffffffu, over)) {
    // ceiling spill (moe_load.py:93-104); rare, done in expert order on the warp
    int64_t sur = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j)
      if (cnt[j] > total) { sur += cnt[j] - total; cnt[j] = total; }
    int64_t surplus = warp_sum_i64(sur);
    for (int jj = 0; jj < E && surplus > 0; ++jj) {
      const int i = (int)order[jj];
      const int owner = i / per, loc = i - owner * per;
      int64_t take = 0;
      if (lane == owner) {
#pragma unroll
        for (int j = 0; j < PER; ++j)
          if (j == loc) {
            const int64_t room = total - cnt[j];
            take = room < surplus ? room : surplus;
            cnt[j] += take;
          }
      }
      take = __shfl_sync(0xffffffffu, take, owner);
      surplus -= take;
    }
  }
}

// busiest contiguous EP block of the counts (expert_shard_tokens + max)
template <int PER>
__device__ __forceinline__ int64_t warp_block_max(const int64_t (&cnt)[PER], int E, int64_t ep) {
  const int lane = threadIdx.x & 31;
  const int per = (E + 31) >> 5;
  // busiest contiguous EP block
  const int bs = (int)(E / ep);
  if (per > 0 && bs % per == 0 && E % 32 == 0 && per * 32 == E) {
    // every lane's experts lie inside one block of bs / per consecutive lanes:
    // segmented warp sum over those lanes, then the maximum over the blocks
    int64_t part = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j)
      if (j < per) part += cnt[j];
    const int lanes = bs / per;  // power of two: E and ep are powers of two here
    if ((lanes & (lanes - 1)) == 0) {
      for (int o = 1; o < lanes && o < 32; o <<= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const int64_t y = __shfl_xor_sync(0xffffffffu, part, o);
        part = y > part ? y : part;
      }
      return part;
    }
  }
  int64_t best = 0;
  for (int r = 0; r < ep; ++r) {
    int64_t part = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int i = lane * per + j;
      if (j < per && i < E && i / bs == r) part += cnt[j];
    }
    const int64_t s = warp_sum_i64(part);
    if (r == 0 || s > best) best = s;
  }
  return best;
}


template <int PER>
__device__ int64_t warp_busiest_shard(const double* __restrict__ q, const double* __restrict__ order, int E,
                                      int64_t total, int64_t topk, int64_t ep, int* hist) {
  int64_t cnt[PER];
  warp_expert_counts<PER>(q, order, E, total, topk, hist, cnt);
  return warp_block_max<PER>(cnt, E, ep);
}

}  // namespace lc
