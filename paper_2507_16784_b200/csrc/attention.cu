// Paged GQA attention over the retained working memory (page size 1).
//
// Reference semantics (model.py:139-159): per layer, queries of the new block
// attend every page of the request's table (the retained prefix, fully
// visible) plus the new block causally; scores = q.k / sqrt(D), softmax with
// max subtraction, ctx = softmax @ V.  The reference has Hq == Hkv; GQA maps
// q head h to kv head h / (Hq/Hkv) (HF repeat_kv convention).
//
// K1 (decode, bf16 KV): persistent stream-K kernel.  The concatenated kv
//   tokens of all decode queries are split evenly over the CTAs, so load is
//   balanced whatever the retained lengths are.  One CTA = 1 producer warp
//   that streams whole page rows (all kv heads of a token: Hkv*D*2 bytes,
//   contiguous in the [layer][page][Hkv][D] pool) into a multi-stage shared
//   ring with TMA bulk copies (cp.async.bulk, SASS UBLKCP) + mbarriers, and
//   Hkv consumer warps (one per kv head) that run QK^T and PV on the tensor
//   cores (mma.sync m16n8k16 bf16, fp32 accumulate) with an online softmax.
//   Queries split across CTAs leave fp32 partials (fire-and-forget stores, no
//   atomic or fence between two stages); after its stream each CTA bumps the
//   arrival counters of its (at most two) split tiles and the last arrival
//   merges the pieces in-kernel (K6, log-sum-exp combine).
//   The same kernel serves extend / re-encode / prefill rows: a work item is
//   a tile of up to 16/group consecutive queries (rows = queries x group
//   heads of the MMA tile) with a causal limit per query.
// Generic (fp32 / any): warp per (row, q head), exact two-pass softmax; used
//   for the fp32 parity configuration.
#include "common.cuh"
#include "attention_tc.cuh"

namespace tim {

constexpr float kLog2e = 1.4426950408889634f;
constexpr int kIdChunk = 512;       // page ids staged per producer refill (multiple of TK)
constexpr int kMinTokensPerCta = 64;  // below this many kv tokens per CTA, use fewer CTAs

// ===================================================================== K1
// HG kv heads per CTA (one page row slice of HG*D*2 contiguous bytes per
// token and layer), WPH consumer warps per kv head (each 16 MMA rows).
// Decode tiles use HG = Hkv, WPH = 1 (one query x all heads, whole 2 KiB page
// rows); multi-token tiles use fewer heads and more warps per head so one
// K/V stream serves WPH x 16/group queries.
#ifndef TIM_RING_BYTES
#define TIM_RING_BYTES 204800   // shared-memory budget of the K/V ring
#endif
template <int D, int HG, int WPH>
struct AttnCfg {
  static constexpr int NW = HG * WPH;                 // consumer warps
  static constexpr int TK = 16;                       // tokens per stage
  static constexpr int ROW_BYTES = HG * D * 2;        // page-row slice per token and layer
  static constexpr int ROW_STRIDE = ROW_BYTES + 16;   // +16B: conflict-free ldmatrix rows
  static constexpr int STAGE_BYTES = 2 * TK * ROW_STRIDE;
  static constexpr int STAGES_RAW = TIM_RING_BYTES / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 12 ? 12 : (STAGES_RAW < 2 ? 2 : STAGES_RAW);
  static constexpr int THREADS = (NW + 2) * 32;        // consumers, producer, publisher
  static constexpr int SMEM = STAGES * STAGE_BYTES + 2 * STAGES * 8 + 16 + kIdChunk * 4 + 16 + 4 * NW + 16;
  static constexpr int KC = D / 16;
  static constexpr int NT = D / 8;
};

// Optional per-CTA timeline (%globaltimer, ns): [start, first data, loop end,
// end, producer stamps, last K6 release, merger count complete] for CTA c at g_trace[8c..8c+7]; enabled by tim_set_trace (diagnostics).
__device__ unsigned long long* g_trace = nullptr;

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int64_t cta_of(int64_t x, int64_t G, int64_t N) {
  return ((x + 1) * G - 1) / N;
}

// Warp-parallel search: the largest r in [0, n) with prefix[r] <= key
// (prefix[0] = 0 <= key).  128 probes per round, all issued before any use,
// so a list of <= 128 tiles costs one memory round trip (the serial binary
// search it replaces cost log2(n) dependent loads at kernel start).
TIM_DEV int seg_search(const int32_t* __restrict__ prefix, int n, int key, int lane) {
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    const int64_t span = hi - lo;
    int32_t v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = __ldg(prefix + lo + (int)(((int64_t)(lane + 32 * j) * span) >> 7));
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) cnt += __popc(__ballot_sync(0xffffffffu, v[j] <= key));
    const int nlo = lo + (int)(((int64_t)(cnt - 1) * span) >> 7);
    hi = cnt < 128 ? lo + (int)(((int64_t)cnt * span) >> 7) : hi;
    lo = nlo;
  }
  return lo;
}

// Tile records of up to 32 consecutive tiles, lane j holding tile rb + j
// (one round trip for the whole batch; fields fetched with shuffles).
struct TileLane {
  int lo, hi, qrow, slot, kv_len, nq, fresh, hgrp;
  TIM_DEV void load(const int32_t* __restrict__ prefix, const int32_t* __restrict__ dec, int n,
                    int rb, int lane) {
    const int r = rb + lane;
    if (r < n) {
      const int32_t* rec = dec + (int64_t)r * TIM_DEC_FIELDS;
      lo = __ldg(prefix + r);
      hi = __ldg(prefix + r + 1);
      qrow = __ldg(rec + 0);
      slot = __ldg(rec + 1);
      kv_len = __ldg(rec + 2);
      nq = __ldg(rec + 3);
      fresh = __ldg(rec + 4);
      hgrp = __ldg(rec + 5);
    } else {
      lo = hi = 0x7fffffff;
      qrow = slot = kv_len = nq = fresh = hgrp = 0;
    }
  }
};
#define TIM_SHFL(v, i) __shfl_sync(0xffffffffu, (v), (i))

TIM_DEV void red_add_release(int32_t* p) {
  asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(p) : "memory");
}
TIM_DEV void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
TIM_DEV int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ------------------------------------------------------------- per-step plan
// The decode-tile partition (G CTAs over N keys) is the same for all layers
// of a step, so tim_attn_plan computes each CTA's first tile once per step
// into the tail of the workspace: int4 header {serial, G, N, 0}, int4 pad,
// then per CTA {start, end, r0, slot0}, {lo0, hi0, fresh0, hgrp0}.  A K1 CTA
// reads its record with the step header (one round trip) instead of a search
// plus a tile-batch load before its first page ids; the record is used only
// when its serial, G and N match the launch (else K1 searches as before).
constexpr int kPlanMaxCtas = 256;
constexpr int kPlanIds = 32;                      // page ids of the CTA's first two stages
constexpr int kPlanRec = 8 + kPlanIds;            // ints per CTA record
constexpr int kPlanInts = 8 + kPlanRec * kPlanMaxCtas;

TIM_DEV int64_t ws_core_floats(int n_ctas, int max_dec, int d) { return (int64_t)(n_ctas + max_dec) * 8 * 16 * (d + 2); }

TIM_DEV const int32_t* plan_of(const float* ws, int n_ctas, int max_dec, int d) {
  return n_ctas <= kPlanMaxCtas ? reinterpret_cast<const int32_t*>(ws + ws_core_floats(n_ctas, max_dec, d)) : nullptr;
}

// CTAs the decode tiles get in the launch that will run them (attn_step_kernel's split logic).
TIM_DEV int dec_grid(const tim_step_header& hd, int n_ctas) {
  if (hd.n_ext == 0) return n_ctas;
  int g0 = hd.split_dec_ctas, g1 = hd.split_ext_ctas;
  if (g0 + g1 <= 0 || g0 + g1 > n_ctas) g0 = hd.n_dec ? n_ctas / 2 : 0;
  return g0;
}

// One warp per CTA record (8 per block): the tile search is the warp-parallel
// seg_search (one round trip for <= 128 tiles) and the record's 32 page ids
// are one load per lane, so the plan costs ~3 dependent round trips whatever
// G is (the single-CTA serial version took 10.6 us per step).
__global__ void __launch_bounds__(256) attn_plan_kernel(const int32_t* __restrict__ step,
                                                        const int32_t* __restrict__ tables, int64_t tstride,
                                                        int n_ctas, int max_dec, int d, float* __restrict__ ws) {
  const tim_step_header& hd = *reinterpret_cast<const tim_step_header*>(step);
  int32_t* plan = reinterpret_cast<int32_t*>(ws + ws_core_floats(n_ctas, max_dec, d));
  const int n_dec = hd.n_dec, N = hd.dec_total;
  const int want = (N + kMinTokensPerCta - 1) / kMinTokensPerCta;
  const int grid = dec_grid(hd, n_ctas);
  const int G = grid < want ? grid : want;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    plan[0] = hd.serial;
    plan[1] = G;
    plan[2] = N;
    plan[3] = 0;
  }
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (n_dec == 0 || N == 0 || c >= G) return;
  const int32_t* dec = step + hd.off_dec;
  const int32_t* prefix = step + hd.off_dec_prefix;
  const int start = (int)((int64_t)c * N / G), end = (int)((int64_t)(c + 1) * N / G);
  const int lo = seg_search(prefix, n_dec, start, lane);
  const int32_t* rec = dec + (int64_t)lo * TIM_DEC_FIELDS;
  const int lo0 = __ldg(prefix + lo), hi0 = __ldg(prefix + lo + 1);
  const int slot = __ldg(rec + 1), fresh = __ldg(rec + 4), hgrp = __ldg(rec + 5);
  int32_t* o = plan + 8 + kPlanRec * c;
  if (lane == 0) {
    reinterpret_cast<int4*>(o)[0] = make_int4(start, end, lo, slot);
    reinterpret_cast<int4*>(o)[1] = make_int4(lo0, hi0, fresh, hgrp);
  }
  // the first page ids of the CTA's piece of that tile (padded with the last)
  const int32_t* trow = tables + (int64_t)slot * tstride;
  const int p0 = start - lo0, n = (end < hi0 ? end : hi0) - lo0 - p0;
  for (int k = lane; k < kPlanIds; k += 32) o[8 + k] = __ldg(trow + p0 + (k < n ? k : n - 1));
}

// Body of K1 for CTA `cta` of the `grid` CTAs that stream the tile list.
template <int D, int HKV, int HG, int WPH>
TIM_DEV void tiles_body(const int32_t* __restrict__ step, int list, const __nv_bfloat16* __restrict__ q,
                        __nv_bfloat16* __restrict__ out, const __nv_bfloat16* __restrict__ kl,
                        const __nv_bfloat16* __restrict__ vl, const int32_t* __restrict__ tables,
                        int64_t tstride, int hq, float scale, float* __restrict__ ws,
                        int32_t* __restrict__ counters, int max_dec, int cta, int grid,
                        const int32_t* __restrict__ plan) {
  using C = AttnCfg<D, HG, WPH>;
  constexpr int NW = C::NW;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  int32_t* s_ids = reinterpret_cast<int32_t*>(empty + C::STAGES);
  uint64_t* pub_bar = reinterpret_cast<uint64_t*>(s_ids + kIdChunk);   // consumers -> publisher
  uint64_t* pub_ack = pub_bar + 1;                                      // publisher read the round
  int32_t* pub_tile = reinterpret_cast<int32_t*>(pub_ack + 1);         // [NW] tile to publish / -1 / -2

  const unsigned long long t_start = gtimer();
  // per-step plan (tim_attn_plan): this CTA's first tile, read in the same
  // round trip as the header instead of searched for afterwards (issued
  // before anything else, the diagnostics pointer included, so the first
  // copies are one round trip away)
  int4 ph = make_int4(0, 0, 0, 0), pa = ph, pb = ph;
  int32_t pid = 0;                           // lane's page id among the first kPlanIds of the range
  if (plan && !list) {
    const int32_t* rec = plan + 8 + kPlanRec * cta;
    ph = __ldg(reinterpret_cast<const int4*>(plan));
    pa = __ldg(reinterpret_cast<const int4*>(rec));
    pb = __ldg(reinterpret_cast<const int4*>(rec) + 1);
    pid = __ldg(rec + 8 + (threadIdx.x & 31));
  }
  const tim_step_header& hd = *reinterpret_cast<const tim_step_header*>(step);
  unsigned long long* trace = g_trace;
  if (trace && threadIdx.x == 0) trace[8 * blockIdx.x] = t_start;
  const int n_dec = list ? hd.n_ext : hd.n_dec;
  const int N = list ? hd.ext_total : hd.dec_total;
  const int want = (N + kMinTokensPerCta - 1) / kMinTokensPerCta;
  const int G = grid < want ? grid : want;
  const int c = cta;
  if (n_dec == 0 || N == 0 || c >= G) {
    // An idle CTA still waits for the preceding grid, so that this grid's
    // completion implies it (the next PDL launch relies on the chain).
    griddep_wait();
    return;
  }
  const int32_t* dec = step + (list ? hd.off_ext : hd.off_dec);
  const int32_t* prefix = step + (list ? hd.off_ext_prefix : hd.off_dec_prefix);
  const int start = (int)((int64_t)c * N / G), end = (int)((int64_t)(c + 1) * N / G);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s2 = 0; s2 < C::STAGES; ++s2) {
      mbar_init(&full[s2], 1);
      mbar_init(&empty[s2], NW);
    }
    mbar_init(pub_bar, NW);
    mbar_init(pub_ack, 1);
    fence_mbar_init();
  }
  // plan record: pa = {start, end, r0, slot0}, pb = {lo0, hi0, fresh0, hgrp0}
  const bool planned = plan && !list && hd.serial != 0 && ph.x == hd.serial && ph.y == G && ph.z == N &&
                       pa.x == start;
  const int r0 = planned ? pa.z : seg_search(prefix, n_dec, start, lane);   // first tile of this CTA
  __syncthreads();
  if (warp > NW + 1) return;   // spare warps of a wider (one-launch) CTA

  if (warp == NW + 1) {
    // ------------------------------------------------------------ publisher
    // Bumps the K6 counters of this CTA's parked partials as soon as the
    // consumer warps hand them over (their stores ordered by the CTA barrier
    // and this warp's gpu-scope release), so a merger in another CTA is not
    // kept waiting for this CTA's stream to end, and no consumer stalls on a
    // release fence.
    for (int round = 0;; ++round) {
      mbar_wait(pub_bar, round & 1);
      const int tile = lane < NW ? pub_tile[lane] : -1;
      __syncwarp();
      if (__all_sync(0xffffffffu, tile == -2 || lane >= NW)) break;
      if (lane == 0) mbar_arrive(pub_ack);   // slots may be rewritten
      if (tile >= 0) red_add_release(counters + (int64_t)tile * 8 + lane);
      if (trace && __any_sync(0xffffffffu, tile >= 0)) {
        __syncwarp();
        if (lane == 0) trace[8 * blockIdx.x + 6] = gtimer();   // last release issued
      }
    }
    return;
  }
  // The tile batch is loaded after the barrier: a planned producer issues its
  // first copies from the plan alone, one round trip after the launch.
  TileLane tl;
  tl.load(prefix, dec, n_dec, r0, lane);

  if (warp == NW) {
    // ------------------------------------------------------------ producer
    // The range is walked as chunks of <= kIdChunk tokens of one tile.  The
    // page ids of chunk k+1 are loaded into registers while chunk k streams,
    // so neither a chunk nor a tile switch puts an id round trip between
    // two stages; each stage is then 2*TK bulk copies of whole page rows.
    const uint64_t pol = l2_evict_first_policy();
    constexpr int IPL = kIdChunk / 32;     // ids per lane
    int32_t idr[IPL];
    int it = 0, rb = r0;
    bool waited = false;
    // chunk cursor: tile r (lane-batch index i), token range [c0, c1) of its piece [.., p1)
    int r = r0, i = 0, c0 = 0, c1 = 0, p1 = 0;
    int slot_cur = 0, fresh_cur = 0, hgrp_cur = 0;
    auto set_range = [&](int lo, int hi) {
      c0 = (start > lo ? start : lo) - lo;
      p1 = (end < hi ? end : hi) - lo;
      c1 = (p1 - c0) < kIdChunk ? p1 : c0 + kIdChunk;
    };
    auto open_tile = [&](int rr) -> bool {     // position the cursor on tile rr's piece
      if (rr >= n_dec) return false;
      if (rr - rb >= 31) {
        rb = rr;
        tl.load(prefix, dec, n_dec, rb, lane);
      }
      const int ii = rr - rb;
      const int lo = TIM_SHFL(tl.lo, ii), hi = TIM_SHFL(tl.hi, ii);
      if (lo >= end) return false;
      r = rr;
      i = ii;
      set_range(lo, hi);
      slot_cur = TIM_SHFL(tl.slot, ii);
      fresh_cur = TIM_SHFL(tl.fresh, ii);
      hgrp_cur = TIM_SHFL(tl.hgrp, ii);
      return true;
    };
    auto fetch = [&]() {                        // ids of the cursor's chunk -> registers
      const int32_t* trow = tables + (int64_t)slot_cur * tstride;
#pragma unroll
      for (int j = 0; j < IPL; ++j) {
        const int k = c0 + lane + 32 * j;
        idr[j] = k < c1 ? __ldg(trow + k) : 0;
      }
    };
    bool more;
    if (planned) {   // first tile straight from the plan: no wait on the tile batch
      set_range(pb.x, pb.y);
      slot_cur = pa.w;
      fresh_cur = pb.z;
      hgrp_cur = pb.w;
      more = true;
    } else {
      more = open_tile(r0);
    }
    if (trace && lane == 0) {
      asm volatile("" ::"r"(slot_cur), "r"(c0));   // stamp once the first tile's fields arrived
      trace[8 * blockIdx.x + 4] = gtimer();
    }
    if (more) fetch();
    // Planned CTAs issue their first two stages straight from the plan's page
    // ids (one per lane), a round trip before the chunk's own id load lands.
    int pre = 0;                                  // keys of the first chunk already issued
    if (planned && more) {
      const int navail = (p1 - c0) < kPlanIds ? (p1 - c0) : kPlanIds;
      for (int k0 = 0; k0 < navail; k0 += C::TK, ++it) {
        const int ntok = (navail - k0) < C::TK ? (navail - k0) : C::TK;
        const int stg = it % C::STAGES;
        if (it >= C::STAGES) mbar_wait(&empty[stg], ((it / C::STAGES) & 1) ^ 1);
        if (!waited && c0 + k0 + ntok > fresh_cur) {
          griddep_wait();
          waited = true;
        }
        const int row = lane & (C::TK - 1);
        const int32_t page = __shfl_sync(0xffffffffu, pid, k0 + (row < ntok ? row : ntok - 1));
#ifdef TIM_CONSUMER_ONLY
        if (lane == 0) mbar_arrive(&full[stg]);
        (void)page;
#else
        if (lane == 0) mbar_arrive_expect_tx(&full[stg], 2 * C::TK * C::ROW_BYTES);
        __syncwarp();
        uint8_t* base = smem + stg * C::STAGE_BYTES + (lane >= C::TK ? C::TK * C::ROW_STRIDE : 0);
        const __nv_bfloat16* src = (lane >= C::TK ? vl : kl) + (int64_t)page * (HKV * D) + (int64_t)hgrp_cur * HG * D;
        bulk_g2s_hint(base + row * C::ROW_STRIDE, src, C::ROW_BYTES, &full[stg], pol);
#endif
        pre = k0 + ntok;
      }
    }
    bool first_chunk = true;
    while (more) {
      __syncwarp();
#pragma unroll
      for (int j = 0; j < IPL; ++j) s_ids[lane + 32 * j] = idr[j];
      if (trace && first_chunk && lane == 0) trace[8 * blockIdx.x + 5] = gtimer();
      __syncwarp();
      const int cur_c0 = c0, cur_c1 = c1;
      const int fresh = fresh_cur;
      const int64_t hoff = (int64_t)hgrp_cur * HG * D;   // head-group slice
      // Advance the cursor and start the next chunk's id loads once this
      // chunk's first stage is out: opening the next tile may wait on the
      // tile batch, which must not delay the first copies of the CTA.
      bool advanced = false;
      auto advance = [&]() {
        if (c1 < p1) {
          c0 = c1;
          c1 = (p1 - c0) < kIdChunk ? p1 : c0 + kIdChunk;
          more = true;
        } else {
          more = open_tile(r + 1);
        }
        if (more) fetch();
        advanced = true;
      };
      for (int k0 = cur_c0 + (first_chunk ? pre : 0); k0 < cur_c1; k0 += C::TK, ++it) {
        const int ntok = (cur_c1 - k0) < C::TK ? (cur_c1 - k0) : C::TK;
        const int stg = it % C::STAGES;
        if (it >= C::STAGES) mbar_wait(&empty[stg], ((it / C::STAGES) & 1) ^ 1);
        // Programmatic dependent launch: pages of earlier tokens were written
        // by earlier steps, so they stream while the preceding RoPE+store
        // kernel still runs; only a stage holding this step's fresh keys
        // (>= the tile's first fresh key) waits for that kernel to finish.
        if (!waited && k0 + ntok > fresh) {
          griddep_wait();
          waited = true;
        }
#ifdef TIM_CONSUMER_ONLY
        if (lane == 0) mbar_arrive(&full[stg]);   // diagnostics: no copies (tools/consumer_only_probe.sh)
        continue;
#endif
        if (lane == 0) mbar_arrive_expect_tx(&full[stg], 2 * C::TK * C::ROW_BYTES);
        __syncwarp();
        const int row = lane & (C::TK - 1);
        const int32_t page = s_ids[k0 - cur_c0 + (row < ntok ? row : ntok - 1)];  // pad rows repeat a valid row
        uint8_t* base = smem + stg * C::STAGE_BYTES + (lane >= C::TK ? C::TK * C::ROW_STRIDE : 0);
        const __nv_bfloat16* src = (lane >= C::TK ? vl : kl) + (int64_t)page * (HKV * D) + hoff;
        bulk_g2s_hint(base + row * C::ROW_STRIDE, src, C::ROW_BYTES, &full[stg], pol);
        if (!advanced) {
          __syncwarp();   // the copies read s_ids: fetch() only fills registers, s_ids is rewritten next chunk
          advance();
        }
      }
      if (!advanced) advance();
      first_chunk = false;
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  griddep_wait();   // q is written by the preceding kernel
  // A work item is a query tile: nq consecutive queries of one request (1 for
  // decode, up to 16/grp for extend / re-encode rows) x the grp q heads of
  // this warp's kv head = the 16 rows of the m16n8k16 tile (row rr = query
  // rr/grp, head rr%grp).  Query qi of the tile sees keys <= kv_len-nq+qi
  // (prefix fully visible, causal inside the new block, model.py:139-140).
  const int grp = hq / HKV;
  const int qpw = 16 / grp;                 // queries per warp (16 MMA rows)
  const int hloc = warp / WPH, sub = warp % WPH;
  const int g = lane >> 2, t = lane & 3;
  const float sl = scale * kLog2e;
  const uint32_t smem_base = smem_u32(smem);
  const int64_t slot_floats = (int64_t)8 * 16 * D;     // one partial: 16 rows x <= 8 warps
  float* ws_o = ws;
  float* ws_ml = ws + (int64_t)(grid + max_dec) * slot_floats;
  int it = 0, rb = r0;
  int pub_round = 0;
  // hand a parked partial's tile (-1: none in this warp, -2: stream done) to
  // the publisher; every consumer warp takes part in every round
  auto publish = [&](int tile) {
    if (pub_round > 0) mbar_wait(pub_ack, (pub_round - 1) & 1);   // previous round read
    __syncwarp();
    if (lane == 0) {
      pub_tile[warp] = tile;
      mbar_arrive(pub_bar);
    }
    ++pub_round;
  };

  // q fragments of a tile for this warp (the A operand of S = Q K^T).  The
  // next tile's fragments are fetched into the same registers as soon as the
  // last QK^T of the current tile has consumed them, so their latency hides
  // behind that stage's softmax / PV and the epilogue (9 warps leave 168
  // registers per thread: no room for a second buffer).
  uint32_t qa[C::KC][4];
  auto load_q = [&](uint32_t (&dst)[C::KC][4], int ii) {
    const int qrow = TIM_SHFL(tl.qrow, ii), nq = TIM_SHFL(tl.nq, ii);
    const int kvh = TIM_SHFL(tl.hgrp, ii) * HG + hloc;
    int nw_q = nq - sub * qpw;
    nw_q = nw_q < 0 ? 0 : (nw_q > qpw ? qpw : nw_q);
    const int nrows = nw_q * grp;
    int orow[2];
    bool valid[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int rr = g + 8 * h;
      valid[h] = rr < nrows;
      orow[h] = (qrow + sub * qpw + rr / grp) * hq + kvh * grp + (rr % grp);
    }
#pragma unroll
    for (int kc = 0; kc < C::KC; ++kc) {
      const int d0 = kc * 16 + 2 * t;
      dst[kc][0] = valid[0] ? *reinterpret_cast<const uint32_t*>(q + (int64_t)orow[0] * D + d0) : 0u;
      dst[kc][1] = valid[1] ? *reinterpret_cast<const uint32_t*>(q + (int64_t)orow[1] * D + d0) : 0u;
      dst[kc][2] = valid[0] ? *reinterpret_cast<const uint32_t*>(q + (int64_t)orow[0] * D + d0 + 8) : 0u;
      dst[kc][3] = valid[1] ? *reinterpret_cast<const uint32_t*>(q + (int64_t)orow[1] * D + d0 + 8) : 0u;
    }
  };
  load_q(qa, 0);

  for (int r = r0; r < n_dec; ++r) {
    if (r - rb == 31) {        // keep tiles r and r + 1 in the lane batch
      rb = r;
      tl.load(prefix, dec, n_dec, rb, lane);
    }
    const int i = r - rb;
    const int lo = TIM_SHFL(tl.lo, i), hi = TIM_SHFL(tl.hi, i);
    if (lo >= end) break;
    const int p0 = (start > lo ? start : lo) - lo;
    const int p1 = (end < hi ? end : hi) - lo;
    const int qrow = TIM_SHFL(tl.qrow, i), kv_len = TIM_SHFL(tl.kv_len, i), nq = TIM_SHFL(tl.nq, i);
    const int kvh = TIM_SHFL(tl.hgrp, i) * HG + hloc;      // this warp's kv head
    int nw_q = nq - sub * qpw;               // queries of this warp in the tile
    nw_q = nw_q < 0 ? 0 : (nw_q > qpw ? qpw : nw_q);
    const int nrows = nw_q * grp;
    const bool has_next = r + 1 < n_dec && TIM_SHFL(tl.lo, i + 1) < end;

    int lim[2], orow[2];
    bool valid[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int rr = g + 8 * h;
      valid[h] = rr < nrows;
      const int qi = sub * qpw + rr / grp;
      lim[h] = kv_len - nq + qi;                          // last visible key (absolute)
      orow[h] = (qrow + qi) * hq + kvh * grp + (rr % grp);
    }

    float o[C::NT][4];
#pragma unroll
    for (int j = 0; j < C::NT; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};

    for (int k0 = p0; k0 < p1; k0 += C::TK, ++it) {
      const int ntok = (p1 - k0) < C::TK ? (p1 - k0) : C::TK;
      const int stg = it % C::STAGES;
      mbar_wait(&full[stg], (it / C::STAGES) & 1);
      if (trace && it == 0 && threadIdx.x == 0) trace[8 * blockIdx.x + 1] = gtimer();
      const uint32_t kbase = smem_base + stg * C::STAGE_BYTES + hloc * D * 2;
      const uint32_t vbase = kbase + C::TK * C::ROW_STRIDE;

      float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
      {
        const int mi = lane >> 3;
        const int tok = (lane & 7) + (mi >> 1) * 8;
        const uint32_t a = kbase + tok * C::ROW_STRIDE + (mi & 1) * 16;
#pragma unroll
        for (int kc = 0; kc < C::KC; ++kc) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4(b0, b1, b2, b3, a + kc * 32);
          mma_bf16(s0, qa[kc][0], qa[kc][1], qa[kc][2], qa[kc][3], b0, b1);
          mma_bf16(s1, qa[kc][0], qa[kc][1], qa[kc][2], qa[kc][3], b2, b3);
        }
      }
      if (has_next && k0 + C::TK >= p1) load_q(qa, i + 1);
      // online softmax (log2 domain); row g -> v[0], row g+8 -> v[1]
      float v[2][4] = {{s0[0], s0[1], s1[0], s1[1]}, {s0[2], s0[3], s1[2], s1[3]}};
      const int tk[4] = {2 * t, 2 * t + 1, 8 + 2 * t, 9 + 2 * t};
      float corr[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float mx = -INFINITY;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          v[h][j] = (tk[j] < ntok && k0 + tk[j] <= lim[h]) ? v[h][j] * sl : -INFINITY;
          mx = fmaxf(mx, v[h][j]);
        }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float mnew = fmaxf(m_r[h], mx);
        const float muse = mnew == -INFINITY ? 0.f : mnew;
        corr[h] = fast_exp2(m_r[h] - muse);
        float sum = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          v[h][j] = fast_exp2(v[h][j] - muse);
          sum += v[h][j];
        }
        l_r[h] = l_r[h] * corr[h] + sum;
        m_r[h] = mnew;
      }
      // Rescale O only when some row's running max moved (warp-uniform test):
      // after the first tiles of a query this is rare, and it is 64 FMULs.
      if (__any_sync(0xffffffffu, corr[0] != 1.f || corr[1] != 1.f)) {
#pragma unroll
        for (int j = 0; j < C::NT; ++j) {
          o[j][0] *= corr[0];
          o[j][1] *= corr[0];
          o[j][2] *= corr[1];
          o[j][3] *= corr[1];
        }
      }
      const uint32_t pa0 = pack_bf16(v[0][0], v[0][1]);
      const uint32_t pa1 = pack_bf16(v[1][0], v[1][1]);
      const uint32_t pa2 = pack_bf16(v[0][2], v[0][3]);
      const uint32_t pa3 = pack_bf16(v[1][2], v[1][3]);
      {
        const int mi = lane >> 3;
        const int tok = (lane & 7) + (mi & 1) * 8;
        const uint32_t a = vbase + tok * C::ROW_STRIDE + (mi >> 1) * 16;
#pragma unroll
        for (int j = 0; j < C::NT / 2; ++j) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(b0, b1, b2, b3, a + j * 32);
          mma_bf16(o[2 * j], pa0, pa1, pa2, pa3, b0, b1);
          mma_bf16(o[2 * j + 1], pa0, pa1, pa2, pa3, b2, b3);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stg]);
    }

    if (trace && threadIdx.x == 0) trace[8 * blockIdx.x + 2] = gtimer();
    // ------------------------------------------------------------ epilogue
    // Per warp, no CTA barrier.  A tile covered by one CTA is written
    // directly.  A split tile is merged (K6) by its designated piece: the one
    // in the tile's first CTA, which is always that CTA's LAST segment, so
    // the merge never stalls a stream.  Every other piece stores its
    // unnormalised partial (O, m, l per row) with fire-and-forget stores and
    // later bumps the (tile, warp) counter with a release reduction; the
    // merger waits for the count, combines the partials with its own
    // registers (its own partial is never written) and re-arms the counter.
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 1);
      l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 2);
    }
    const int cf = (int)cta_of(lo, G, N), cl = (int)cta_of(hi - 1, G, N);
    if (cf != cl && c != cf) {
      // non-merger piece: park the partial and hand it to the publisher warp
      const int64_t wslot = ((int64_t)(c + r) * 8 + warp) * 16;   // first of this warp's 16 partial rows
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rr = g + 8 * h;
        if (valid[h]) {
          float* ob = ws_o + (wslot + rr) * D;
#pragma unroll
          for (int j = 0; j < C::NT; ++j)
            __stcg(reinterpret_cast<float2*>(ob + j * 8 + 2 * t), make_float2(o[j][2 * h], o[j][2 * h + 1]));
          if (t == 0) __stcg(reinterpret_cast<float2*>(ws_ml + (wslot + rr) * 2), make_float2(m_r[h], l_r[h]));
        }
      }
      publish(nrows > 0 ? r : -1);
      continue;
    }
    if (cf != cl && nrows > 0) {
      // merger (this CTA's last segment): wait for the other pieces
      int32_t* cnt = counters + (int64_t)r * 8 + warp;
      // Pull the other pieces' partials toward L2 while waiting: they were
      // parked up to a whole launch earlier and are mostly evicted by the
      // stream by now, and the merge below sits on the kernel's tail (L2 is
      // the coherence point, so fetching a line before its final write is
      // harmless).
      for (int p = cf + 1; p <= cl; ++p) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (!valid[h]) continue;
          const int64_t wrow = ((int64_t)(p + r) * 8 + warp) * 16 + g + 8 * h;
          prefetch_l2(ws_o + wrow * D + 32 * t);
          if (t == 0) prefetch_l2(ws_ml + wrow * 2);
        }
      }
      // Lane 0 acquires the count; the warp barrier orders the other lanes'
      // partial loads after it (they read through L2, .cg, where the
      // publishers' released stores live), saving a second round trip.
      if (lane == 0) {
        while (ld_acquire(cnt) < cl - cf) {
        }
        *cnt = 0;   // re-arm for the next launch
        if (trace && warp == 0) trace[8 * blockIdx.x + 7] = gtimer();   // merger's count complete
      }
      __syncwarp();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rr = g + 8 * h;
        if (!valid[h]) continue;
        for (int p = cf + 1; p <= cl; ++p) {
          const int64_t wrow = ((int64_t)(p + r) * 8 + warp) * 16 + rr;
          const float2 ml = __ldcg(reinterpret_cast<const float2*>(ws_ml + wrow * 2));
          const float* ob = ws_o + wrow * D;
          float2 op[C::NT];
#pragma unroll
          for (int j = 0; j < C::NT; ++j) op[j] = __ldcg(reinterpret_cast<const float2*>(ob + j * 8 + 2 * t));
          const float mm = fmaxf(m_r[h], ml.x);
          const float sa = m_r[h] == -INFINITY ? 0.f : fast_exp2(m_r[h] - mm);
          const float sb = ml.x == -INFINITY ? 0.f : fast_exp2(ml.x - mm);
#pragma unroll
          for (int j = 0; j < C::NT; ++j) {
            o[j][2 * h] = o[j][2 * h] * sa + op[j].x * sb;
            o[j][2 * h + 1] = o[j][2 * h + 1] * sa + op[j].y * sb;
          }
          l_r[h] = l_r[h] * sa + ml.y * sb;
          m_r[h] = mm;
        }
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (valid[h]) {
        const float inv = 1.f / l_r[h];
        __nv_bfloat16* ob = out + (int64_t)orow[h] * D;
#pragma unroll
        for (int j = 0; j < C::NT; ++j)
          *reinterpret_cast<uint32_t*>(ob + j * 8 + 2 * t) =
              pack_bf16(o[j][2 * h] * inv, o[j][2 * h + 1] * inv);
      }
    }
  }
  publish(-2);   // the publisher warp may retire
  if (trace && threadIdx.x == 0) trace[8 * blockIdx.x + 3] = gtimer();
}

template <int D, int HKV, int HG, int WPH>
__global__ void __launch_bounds__(AttnCfg<D, HG, WPH>::THREADS, 1)
    attn_tiles_kernel(const int32_t* __restrict__ step, int list, const __nv_bfloat16* __restrict__ q,
                      __nv_bfloat16* __restrict__ out, const __nv_bfloat16* __restrict__ kl,
                      const __nv_bfloat16* __restrict__ vl, const int32_t* __restrict__ tables,
                      int64_t tstride, int hq, float scale, float* __restrict__ ws,
                      int32_t* __restrict__ counters, int max_dec) {
  griddep_launch();   // let the next kernel get resident early
  tiles_body<D, HKV, HG, WPH>(step, list, q, out, kl, vl, tables, tstride, hq, scale, ws, counters, max_dec,
                              blockIdx.x, gridDim.x, plan_of(ws, gridDim.x, max_dec, D));
}

__global__ void __launch_bounds__(tc::THREADS, 1)
    attn_ext_tc_kernel(const __nv_bfloat16* __restrict__ kl, const __nv_bfloat16* __restrict__ vl,
                       const int32_t* __restrict__ step, const __nv_bfloat16* __restrict__ q,
                       __nv_bfloat16* __restrict__ out, const int32_t* __restrict__ tables,
                       int64_t tstride, int hq, int hkv, float scale_log2) {
  griddep_launch();
  ext_tc_body(kl, vl, step, q, out, tables, tstride, hq, hkv, scale_log2, blockIdx.x, gridDim.x);
}

// One launch for a whole step's attention (decode tiles + multi-token items):
// the first split_dec_ctas CTAs stream the decode tiles (K1), the others work
// the tcgen05 items (K2), concurrently, with the split the host derived from
// the two lists' work (tim_step_header.split_*).  Keeps programmatic
// dependent launch after the RoPE/store kernel, which two launches on forked
// streams would lose.
template <int D, int HKV>
constexpr int step_threads() {
  return AttnCfg<D, HKV, 1>::THREADS > tc::THREADS ? AttnCfg<D, HKV, 1>::THREADS : tc::THREADS;
}

template <int D, int HKV>
__global__ void __launch_bounds__(step_threads<D, HKV>(), 1)
    attn_step_kernel(const int32_t* __restrict__ step, const __nv_bfloat16* __restrict__ q,
                     __nv_bfloat16* __restrict__ out, const __nv_bfloat16* __restrict__ kl,
                     const __nv_bfloat16* __restrict__ vl, const int32_t* __restrict__ tables,
                     int64_t tstride, int hq, float scale, float* __restrict__ ws,
                     int32_t* __restrict__ counters, int max_dec) {
  griddep_launch();
  const tim_step_header& hd = *reinterpret_cast<const tim_step_header*>(step);
  int g0 = hd.split_dec_ctas, g1 = hd.split_ext_ctas;
  if (g0 + g1 <= 0 || g0 + g1 > (int)gridDim.x) {   // no split planned by the host
    g0 = hd.n_ext ? (hd.n_dec ? (int)gridDim.x / 2 : 0) : (int)gridDim.x;
    g1 = gridDim.x - g0;
  }
  const int c = blockIdx.x;
  if (c < g0)
    tiles_body<D, HKV, HKV, 1>(step, 0, q, out, kl, vl, tables, tstride, hq, scale, ws, counters, max_dec, c, g0,
                               plan_of(ws, gridDim.x, max_dec, D));
  else if (c < g0 + g1) {
    const unsigned long long t0 = gtimer();
    ext_tc_body(kl, vl, step, q, out, tables, tstride, hq, HKV, scale * kLog2e, c - g0, g1);
    if (g_trace && threadIdx.x == 0) {   // diagnostics: K2 CTA start / end in the K1 slot layout
      g_trace[8 * c] = t0;
      g_trace[8 * c + 3] = gtimer();
    }
  } else
    griddep_wait();
}

// ================================================================ generic
// Warp per (row, q head); exact two-pass softmax in fp32 (model.py:154-159).
template <typename T>
__global__ void attn_generic_kernel(const int32_t* __restrict__ step, const T* __restrict__ q,
                                    T* __restrict__ out, const T* __restrict__ kl,
                                    const T* __restrict__ vl, const int32_t* __restrict__ tables,
                                    int64_t tstride, int hq, int hkv, int D, float scale) {
  const tim_step_header& hd = *reinterpret_cast<const tim_step_header*>(step);
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int row = wid / hq, head = wid - row * hq;
  if (row >= hd.n_rows) return;
  const int32_t* segs = step + hd.off_segs;
  int lo = 0, hi = hd.n_segs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (segs[mid * TIM_SEG_FIELDS + 3] <= row) lo = mid; else hi = mid - 1;
  }
  const int slot = segs[lo * TIM_SEG_FIELDS], m = segs[lo * TIM_SEG_FIELDS + 1];
  const int i = row - segs[lo * TIM_SEG_FIELDS + 3];
  const int kv_len = m + i + 1;  // prefix fully visible + causal within the new block
  const int kvh = head / (hq / hkv);
  const int32_t* trow = tables + (int64_t)slot * tstride;
  constexpr int MAXE = 8;  // D <= 256
  float qv[MAXE], ov[MAXE];
  const T* qp = q + ((int64_t)row * hq + head) * D;
#pragma unroll
  for (int k = 0; k < MAXE; ++k) {
    const int e = lane + 32 * k;
    qv[k] = e < D ? to_f32(qp[e]) : 0.f;
    ov[k] = 0.f;
  }
  float mx = -INFINITY;
  for (int j = 0; j < kv_len; ++j) {
    const T* kp = kl + ((int64_t)trow[j] * hkv + kvh) * D;
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < MAXE; ++k) {
      const int e = lane + 32 * k;
      if (e < D) acc += qv[k] * to_f32(kp[e]);
    }
    mx = fmaxf(mx, warp_sum(acc) * scale);
  }
  float den = 0.f;
  for (int j = 0; j < kv_len; ++j) {
    const int64_t pg = trow[j];
    const T* kp = kl + (pg * hkv + kvh) * D;
    const T* vp = vl + (pg * hkv + kvh) * D;
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < MAXE; ++k) {
      const int e = lane + 32 * k;
      if (e < D) acc += qv[k] * to_f32(kp[e]);
    }
    const float w = expf(warp_sum(acc) * scale - mx);
    den += w;
#pragma unroll
    for (int k = 0; k < MAXE; ++k) {
      const int e = lane + 32 * k;
      if (e < D) ov[k] += w * to_f32(vp[e]);
    }
  }
  T* op = out + ((int64_t)row * hq + head) * D;
#pragma unroll
  for (int k = 0; k < MAXE; ++k) {
    const int e = lane + 32 * k;
    if (e < D) op[e] = from_f32<T>(ov[k] / den);
  }
}

// Split tiles are merged by a CTA that spins on the other pieces' counter
// (K6).  That is deadlock-free only if every CTA of the grid can be resident at
// once: a dependent grid can start only after every CTA of this one has run
// its griddepcontrol.launch_dependents (the first instruction), i.e. is already
// resident, so nothing launched later takes a slot a waited-on CTA needs.
// Refuse a grid larger than the device's co-residency capacity for the
// kernel's threads and shared memory.
template <class Kern>
int32_t check_coresident(Kern kern, int threads, int smem, int n_ctas, int* cap, const char* name) {
  if (*cap <= 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    *cap = per_sm * sms;
  }
  if (n_ctas > *cap) {
    set_last_error("%s: grid of %d CTAs exceeds the %d co-resident CTAs the split-tile merge needs",
                   name, n_ctas, *cap);
    return TIM_BAD_ARGUMENT;
  }
  return TIM_OK;
}

template <int D, int HKV, int HG, int WPH>
int32_t launch_tiles(const int32_t* step, int list, const void* q, void* out, const void* kl,
                     const void* vl, const int32_t* tables, int64_t tstride, int hq, float scale,
                     float* ws, int32_t* counters, int n_ctas, int max_dec, cudaStream_t st) {
  using C = AttnCfg<D, HG, WPH>;
  auto kern = attn_tiles_kernel<D, HKV, HG, WPH>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  static int cap = 0;
  if (const int32_t rc = check_coresident(kern, C::THREADS, C::SMEM, n_ctas, &cap, "attn_tiles")) return rc;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_ctas);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, step, list, (const __nv_bfloat16*)q,
                                           (__nv_bfloat16*)out, (const __nv_bfloat16*)kl,
                                           (const __nv_bfloat16*)vl, tables, tstride, hq, scale,
                                           ws, counters, max_dec);
  if (e != cudaSuccess) {
    set_last_error("attn_tiles launch: %s", cudaGetErrorString(e));
    return TIM_CUDA_ERROR;
  }
  return check_launch("attn_tiles");
}

bool ext_tc_shape(int hq, int hkv, int head_dim) {
  return head_dim == tc::D && hkv > 0 && hq == tc::GRP * hkv;
}

int32_t launch_ext_tc(const int32_t* step, const void* q, void* out, const void* kl, const void* vl,
                      const int32_t* tables, int64_t tstride, int hq, int hkv, float scale,
                      int n_ctas, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_ext_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM);
    attr = true;
  }
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_ctas);
  cfg.blockDim = dim3(tc::THREADS);
  cfg.dynamicSmemBytes = tc::SMEM;
  cfg.stream = st;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, attn_ext_tc_kernel, (const __nv_bfloat16*)kl,
                                           (const __nv_bfloat16*)vl, step, (const __nv_bfloat16*)q,
                                           (__nv_bfloat16*)out, tables, tstride, hq, hkv, scale * kLog2e);
  if (e != cudaSuccess) {
    set_last_error("attn_ext_tc launch: %s", cudaGetErrorString(e));
    return TIM_CUDA_ERROR;
  }
  return check_launch("attn_ext_tc");
}

template <int D, int HKV>
int32_t launch_step(const int32_t* step, const void* q, void* out, const void* kl, const void* vl,
                    const int32_t* tables, int64_t tstride, int hq, float scale, float* ws, int32_t* counters,
                    int n_ctas, int max_dec, cudaStream_t st) {
  constexpr int SMEM = AttnCfg<D, HKV, 1>::SMEM > tc::SMEM ? AttnCfg<D, HKV, 1>::SMEM : tc::SMEM;
  auto kern = attn_step_kernel<D, HKV>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    attr = true;
  }
  static int cap = 0;
  if (const int32_t rc = check_coresident(kern, step_threads<D, HKV>(), SMEM, n_ctas, &cap, "attn_step"))
    return rc;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_ctas);
  cfg.blockDim = dim3(step_threads<D, HKV>());
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = st;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, step, (const __nv_bfloat16*)q, (__nv_bfloat16*)out,
                                           (const __nv_bfloat16*)kl, (const __nv_bfloat16*)vl, tables, tstride,
                                           hq, scale, ws, counters, max_dec);
  if (e != cudaSuccess) {
    set_last_error("attn_step launch: %s", cudaGetErrorString(e));
    return TIM_CUDA_ERROR;
  }
  return check_launch("attn_step");
}

// kv heads per CTA for multi-token tiles (the rest of the 8 warps share a head)
constexpr int ext_hg(int hkv) { return hkv >= 8 ? 4 : (hkv >= 4 ? 2 : 1); }

}  // namespace tim

using namespace tim;

static bool tensor_core_shape(int32_t hq, int32_t hkv, int32_t head_dim) {
  if (hkv <= 0 || hq % hkv) return false;
  const int grp = hq / hkv;
  const bool grp_ok = grp == 1 || grp == 2 || grp == 4 || grp == 8 || grp == 16;
  const bool hkv_ok = hkv == 1 || hkv == 2 || hkv == 4 || hkv == 8;
  return grp_ok && hkv_ok && (head_dim == 64 || head_dim == 128);
}

extern "C" int64_t tim_decode_ws_floats(int32_t n_ctas, int32_t max_dec, int32_t hkv, int32_t head_dim) {
  (void)hkv;  // partial slots are sized for the 8 consumer warps of a CTA; the plan follows them
  return (int64_t)(n_ctas + max_dec) * 8 * 16 * (head_dim + 2) + kPlanInts;
}

extern "C" int32_t tim_attn_plan(const int32_t* step, const int32_t* block_tables, int64_t table_stride,
                                 int32_t n_ctas, int32_t max_dec, int32_t head_dim, float* ws, void* stream) {
  if (n_ctas <= 0 || n_ctas > kPlanMaxCtas) return TIM_OK;   // K1 falls back to its own search
  prefer_shared(attn_plan_kernel);
  attn_plan_kernel<<<(n_ctas + 7) / 8, 256, 0, (cudaStream_t)stream>>>(step, block_tables, table_stride,
                                                                       n_ctas, max_dec, head_dim, ws);
  return check_launch("attn_plan");
}

extern "C" int32_t tim_extend_queries_per_item(int32_t hq, int32_t hkv, int32_t head_dim, int32_t dtype) {
  // queries per multi-token attention tile (mode 1 of tim_attn_decode)
  if (dtype == TIM_DTYPE_BF16 && ext_tc_shape(hq, hkv, head_dim)) return tc::QBLK * tc::M / (hq / hkv);
  if (dtype == TIM_DTYPE_BF16 && tensor_core_shape(hq, hkv, head_dim))
    return (8 / ext_hg(hkv)) * (16 / (hq / hkv));
  return 1 << 30;  // generic path: whole segments
}

extern "C" int32_t tim_extend_head_groups(int32_t hq, int32_t hkv, int32_t head_dim) {
  if (ext_tc_shape(hq, hkv, head_dim)) return hkv;   // one tcgen05 item per kv head
  return hkv / ext_hg(hkv);
}

static int32_t launch_generic(const int32_t* step, int32_t n_rows, const void* q, void* out,
                              const void* kl, const void* vl, const int32_t* tables,
                              int64_t tstride, int32_t hq, int32_t hkv, int32_t D, float scale,
                              int32_t dtype, cudaStream_t st) {
  if (D > 256) { set_last_error("head_dim > 256 unsupported"); return TIM_UNSUPPORTED; }
  const int64_t warps = (int64_t)n_rows * hq;
  const int blocks = (int)((warps * 32 + 255) / 256);
  if (blocks <= 0) return TIM_OK;
  if (dtype == TIM_DTYPE_F32) {
    attn_generic_kernel<float><<<blocks, 256, 0, st>>>(step, (const float*)q, (float*)out,
                                                       (const float*)kl, (const float*)vl, tables,
                                                       tstride, hq, hkv, D, scale);
  } else {
    attn_generic_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(
        step, (const __nv_bfloat16*)q, (__nv_bfloat16*)out, (const __nv_bfloat16*)kl,
        (const __nv_bfloat16*)vl, tables, tstride, hq, hkv, D, scale);
  }
  return check_launch("attn_generic");
}

// Rows handled: decode queries listed in the step (n_dec).  For the fp32 /
// generic configuration every row is handled by tim_attn_extend instead.
extern "C" int32_t tim_attn_decode(const int32_t* step, int32_t mode, const void* q, void* out,
                                   const void* k_layer, const void* v_layer,
                                   const int32_t* block_tables, int64_t table_stride, int32_t hq,
                                   int32_t hkv, int32_t head_dim, float scale, float* ws,
                                   int32_t* counters, int32_t n_ctas, int32_t max_dec,
                                   int32_t dtype, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype != TIM_DTYPE_BF16 || !tensor_core_shape(hq, hkv, head_dim)) {
    set_last_error("tim_attn_decode: tensor-core path needs bf16, hkv in {1,2,4,8}, "
                   "group in {1,2,4,8,16}, D in {64,128}");
    return TIM_UNSUPPORTED;
  }
  if (n_ctas <= 0) return TIM_OK;
#define TIM_TILES(DD, HH)                                                                      \
  if (head_dim == DD && hkv == HH) {                                                           \
    if (mode == 0)                                                                             \
      return launch_tiles<DD, HH, HH, 1>(step, 0, q, out, k_layer, v_layer, block_tables,      \
                                         table_stride, hq, scale, ws, counters, n_ctas, max_dec, st); \
    return launch_tiles<DD, HH, ext_hg(HH), 8 / ext_hg(HH)>(step, 1, q, out, k_layer, v_layer, \
                                                            block_tables, table_stride, hq,    \
                                                            scale, ws, counters, n_ctas, max_dec, st); \
  }
  if (mode == 2) {   // the step's decode tiles and multi-token items in one launch
    if (head_dim == 128 && hkv == 8 && ext_tc_shape(hq, hkv, head_dim))
      return launch_step<128, 8>(step, q, out, k_layer, v_layer, block_tables, table_stride, hq, scale, ws,
                                 counters, n_ctas, max_dec, st);
    const int32_t e0 = tim_attn_decode(step, 0, q, out, k_layer, v_layer, block_tables, table_stride, hq,
                                       hkv, head_dim, scale, ws, counters, n_ctas, max_dec, dtype, stream);
    if (e0 != TIM_OK) return e0;
    mode = 1;
  }
  if (mode == 1 && ext_tc_shape(hq, hkv, head_dim))   // multi-token tiles on tcgen05 (attention_tc.cuh)
    return launch_ext_tc(step, q, out, k_layer, v_layer, block_tables, table_stride, hq, hkv, scale,
                         n_ctas, st);
  TIM_TILES(128, 8) TIM_TILES(128, 4) TIM_TILES(128, 2) TIM_TILES(128, 1)
  TIM_TILES(64, 8) TIM_TILES(64, 4) TIM_TILES(64, 2) TIM_TILES(64, 1)
#undef TIM_TILES
  return TIM_UNSUPPORTED;
}

extern "C" int32_t tim_attn_extend(const int32_t* step, int32_t max_items, const void* q, void* out,
                                   const void* k_layer, const void* v_layer,
                                   const int32_t* block_tables, int64_t table_stride, int32_t hq,
                                   int32_t hkv, int32_t head_dim, float scale, int32_t dtype,
                                   void* stream) {
  // Reference-precision path (fp32, or shapes outside the tensor-core
  // kernel): every row of the step's segments; max_items bounds the rows.
  if (max_items <= 0) return TIM_OK;
  return launch_generic(step, max_items, q, out, k_layer, v_layer, block_tables, table_stride, hq,
                        hkv, head_dim, scale, dtype, (cudaStream_t)stream);
}

extern "C" int32_t tim_tc_trace(void* buf) {
  unsigned long long* p = (unsigned long long*)buf;
  if (cudaMemcpyToSymbol(tim::g_tc_trace, &p, sizeof(p)) != cudaSuccess) return TIM_CUDA_ERROR;
  return TIM_OK;
}

extern "C" int32_t tim_set_trace(void* buf) {
  unsigned long long* p = (unsigned long long*)buf;
  const cudaError_t e = cudaMemcpyToSymbol(tim::g_trace, &p, sizeof(p));
  if (e != cudaSuccess) {
    tim::set_last_error("set_trace: %s", cudaGetErrorString(e));
    return TIM_CUDA_ERROR;
  }
  return TIM_OK;
}
