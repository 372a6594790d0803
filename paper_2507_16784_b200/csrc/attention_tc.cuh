// Included by attention.cu (one translation unit, so the single-launch step
// kernel can host both bodies).
#pragma once
// K2 on the 5th-gen tensor cores: attention of the multi-token rows of a step
// (re-encoded suffixes after a prune, tool responses, prefills) over their
// paged prefix + causal new block (model.py:139-159).
//
// Why a separate kernel: the decode kernel (attention.cu, mma.sync) streams
// whole page rows for 4 queries per tile, so a 150-row re-encode re-reads its
// ~700-token prefix ~38 times, and its per-warp m16n8k16 chains are latency
// bound (ncu: HMMA pipe <20 % busy, consumers starved on a 3-stage ring).  Here
// one work item is 64 queries x the 4 q heads of one kv head = two q-blocks of
// 128 MMA rows that share every K/V block, so each kv head's K/V slice is
// streamed once per 64 queries, and S = Q K^T / O += P V are single-thread
// tcgen05.mma issues (M=128, N=64 / N=128 per q-block) with fp32 accumulators
// in TMEM (all 512 columns).
//
// Per CTA (persistent, one per SM, items round-robin):
//   warp 9     producer: page ids -> 16-byte cp.async of the kv head's 256-byte
//              K and V rows into a 3-stage ring of 64-token blocks, stored
//              128B-swizzled, i.e. the canonical UMMA layouts (K: K-major B
//              operand, V: MN-major B).  (TMA tile::gather4 does the same with
//              128-byte rows but was measured ~10x slower per byte here.)
//   warp 8     MMA issuer (one thread): S_j = Q K_j^T into one of two TMEM S
//              buffers per q-block, O += P_j V_j into the q-block's O.
//   warps 0-7  softmax / epilogue, warps 4b..4b+3 own q-block b; thread t <->
//              TMEM lane t <-> MMA row t of its q-block (query t/4, head t%4 of
//              the kv head): tcgen05.ld of its 64
//              scores, causal mask, online softmax in the log2 domain with
//              lazy rescaling (O is rescaled in TMEM only when the running max
//              grows by more than 2^8), P as bf16 into a swizzled smem tile
//              (the A operand of the PV MMA); at the end O / l -> bf16 -> out.
#include "common.cuh"

namespace tim {
namespace tc {

constexpr int D = 128;               // head dim (two 64-element, 128-byte slabs)
constexpr int GRP = 4;               // q heads per kv head
constexpr int M = 128;               // MMA rows per item
constexpr int BN = 64;               // keys per block
constexpr int QBLK = 2;              // q-blocks per item: two MMA row tiles share each K/V block
constexpr int ST = 5;                // K/V ring stages
constexpr int Q_SLAB = M * 128;      // 16 KiB
constexpr int Q_BYTES = 2 * Q_SLAB;  // 32 KiB
constexpr int P_BYTES = M * 128;     // 16 KiB (128 rows x 64 keys bf16)
constexpr int KV_SLAB = BN * 128;    // 8 KiB (64 keys x 64 elements)
constexpr int K_BYTES = 2 * KV_SLAB;
constexpr int STAGE = 2 * K_BYTES;   // K then V, 32 KiB
constexpr int BAR_BYTES = 256;
constexpr int SMEM = 1024 + QBLK * Q_BYTES + ST * STAGE + BAR_BYTES;
constexpr int THREADS = 10 * 32;     // 8 softmax warps (4 per q-block), MMA, producer
constexpr int MMA_WARP = 8, PROD_WARP = 9;
constexpr int TMEM_COLS = 512;       // S[2 buffers][2 q-blocks] (64 cols each) + O[2 q-blocks] (128 cols)
constexpr uint32_t O_COL = 256;
constexpr float kRescaleLog2 = 8.f;  // lazy rescale threshold (p <= 2^8 with a stale max)

// kind::f16 instruction descriptors (bf16 x bf16 -> f32, M = 128)
constexpr uint32_t kIdescS = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(M >> 4) << 24);                       // B = K, K-major
constexpr uint32_t kIdescO = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                             ((uint32_t)(D >> 3) << 17) | ((uint32_t)(M >> 4) << 24);  // B = V, MN-major

// UMMA smem descriptor, 128B swizzle, SM100 version bit.  K-major: 8-row
// groups 1024 B apart (SBO); MN-major: 8 K-rows 1024 B apart (SBO), 64-element
// MN atoms LBO apart.
TIM_DEV uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}

TIM_DEV void mma_ss(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// D += A * B with A (M x 16, bf16, K-major) read from TMEM: the P tile the
// softmax stored over its S buffer (lane = row, 2 bf16 per 32-bit column).
TIM_DEV void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
TIM_DEV void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
TIM_DEV void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
TIM_DEV void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

TIM_DEV void tld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
TIM_DEV void tst32(uint32_t taddr, const float (&v)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};"
               ::"r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])), "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])), "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])), "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])), "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])), "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
               : "memory");
}
TIM_DEV bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
TIM_DEV void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
// ex2.approx without `volatile`, so the compiler may interleave the 64
// exponentials of a row with the surrounding FMA-pipe work
TIM_DEV float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
TIM_DEV void tld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
TIM_DEV void tst_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// byte offset of 16-byte chunk c (0..7) of row r in a 128B-swizzled slab
TIM_DEV uint32_t swz(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

}  // namespace tc

using namespace tc;

// Diagnostics: per-block %globaltimer stamps of CTA 0 (tim_tc_trace).
static __device__ unsigned long long* g_tc_trace = nullptr;
TIM_DEV unsigned long long tc_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TCT(slot, g) do { if (tr && (g) < 64) tr[(g) * 8 + (slot)] = tc_now(); } while (0)

// Body of the multi-token kernel for CTA `cta` of `grid` CTAs working the
// step's ext list (warps >= 6 of a wider CTA only take part in the barriers).
TIM_DEV void ext_tc_body(const __nv_bfloat16* __restrict__ kl, const __nv_bfloat16* __restrict__ vl,
                         const int32_t* __restrict__ step, const __nv_bfloat16* __restrict__ q,
                         __nv_bfloat16* __restrict__ out, const int32_t* __restrict__ tables,
                         int64_t tstride, int hq, int hkv, float scale_log2, int cta, int grid) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                       // [q-block] 32 KiB A tiles
  uint8_t* sKV = sQ + QBLK * Q_BYTES;
  uint64_t* kv_full = reinterpret_cast<uint64_t*>(sKV + ST * STAGE);
  uint64_t* kv_empty = kv_full + ST;
  uint64_t* s_ready = kv_empty + ST;   // [2]
  uint64_t* p_ready = s_ready + 2;     // [2]
  uint64_t* pv_done = p_ready + 2;     // [2]
  uint64_t* q_ready = pv_done + 2;     // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_ready + 1);

  unsigned long long* tr = cta == 0 ? g_tc_trace : nullptr;
  const tim_step_header& hd = *reinterpret_cast<const tim_step_header*>(step);
  const int n_items = hd.n_ext;
  if (n_items == 0 || cta >= n_items) {
    griddep_wait();   // completion of this grid must imply the preceding one's
    return;
  }
  const int32_t* items = step + hd.off_ext;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&kv_full[s], 32);
      mbar_init(&kv_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_ready[b], 1);
      mbar_init(&p_ready[b], QBLK * M);
      mbar_init(&pv_done[b], 1);
    }
    mbar_init(q_ready, QBLK * M);
    fence_mbar_init();
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)), "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == PROD_WARP) {
    // ---------------------------------------------------------- producer
    // 16-byte cp.async (LDGSTS) of the kv head's 256-byte K and V rows into
    // the swizzled slabs: a warp instruction moves two whole rows, where a TMA
    // gather4 moves four 128-byte rows per (much slower) TMA request.  Each
    // lane's copies of a block complete onto the block's barrier
    // (cp.async.mbarrier.arrive.noinc), so publication never waits on issue;
    // the MMA thread fences the async proxy before the tensor cores read it.
    bool waited = false;
    int gb = 0;
    const int ch = lane & 15, tsub = lane >> 4;     // 16-byte chunk of a row, token parity
    for (int it = cta; it < n_items; it += grid) {
      const int32_t* rec = items + (int64_t)it * TIM_EXT_FIELDS;
      const int slot = rec[1], kv_len = rec[2], fresh = rec[4], head = rec[5];
      const int32_t* trow = tables + (int64_t)slot * tstride;
      const int nblk = (kv_len + BN - 1) / BN;
      for (int j = 0; j < nblk; ++j, ++gb) {
        const int k0 = j * BN;
        const int stg = gb % ST;
        int pid[2];
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          int k = k0 + lane + 32 * h2;
          if (k >= kv_len) k = kv_len - 1;           // pad keys repeat a valid row (masked)
          pid[h2] = __ldg(trow + k);
        }
        if (gb >= ST) mbar_wait(&kv_empty[stg], ((gb / ST) & 1) ^ 1);
        if (lane == 0) TCT(0, gb);
        // keys >= fresh were written by the preceding RoPE/store kernel
        if (!waited && k0 + BN > fresh) {
          griddep_wait();
          waited = true;
        }
        uint8_t* kd = sKV + stg * STAGE;
#pragma unroll
        for (int i = 0; i < BN / 2; ++i) {
          const int tok = 2 * i + tsub;
          const int page = __shfl_sync(0xffffffffu, pid[i >> 4], tok & 31);
          const int64_t src = ((int64_t)page * hkv + head) * D + ch * 8;
          const uint32_t doff = (ch >> 3) * KV_SLAB + swz(tok, ch & 7);
          cp_async16(kd + doff, kl + src);
          cp_async16(kd + K_BYTES + doff, vl + src);
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&kv_full[stg]))
                     : "memory");
      }
    }
    cp_async_wait<0>();
  } else if (warp == MMA_WARP) {
    // ---------------------------------------------------------- MMA issuer
    // Event loop over two cursors: the next S_g = Q K_g^T (needs its K block
    // and its item's Q, and S buffer g&1 released, i.e. PV_{g-2} issued) and
    // the next O += P_g V_g (needs the softmax's P_g).  Whichever is ready is
    // issued, so neither waits behind the other's data.
    if (lane == 0) {
      const uint32_t qa = smem_u32(sQ), kva = smem_u32(sKV);
      auto nblk_of = [&](int it) {
        return it < n_items ? (items[(int64_t)it * TIM_EXT_FIELDS + 2] + BN - 1) / BN : 0;
      };
      auto nqb_of = [&](int it) {   // q-blocks holding queries (an item of <= 32 queries has one)
        return it < n_items ? (items[(int64_t)it * TIM_EXT_FIELDS + 3] + M / GRP - 1) / (M / GRP) : 0;
      };
      int s_it = cta, s_j = 0, s_g = 0, s_ii = 0, s_nb = nblk_of(s_it), s_nqb = nqb_of(s_it);
      int p_it = cta, p_j = 0, p_g = 0, p_nb = s_nb, p_nqb = s_nqb;
      bool q_ok = false;
      while (p_it < n_items) {
        bool progress = false;
        if (s_it < n_items && s_g <= p_g + 1) {
          if (!q_ok && mbar_test(q_ready, s_ii & 1)) q_ok = true;
          const int stg = s_g % ST;
          if (q_ok && mbar_test(&kv_full[stg], (s_g / ST) & 1)) {
            TCT(2, s_g);
            fence_proxy_async();          // cp.async (generic proxy) data -> tensor-core reads
            fence_after();
            const uint32_t kb = kva + stg * STAGE;
#pragma unroll
            for (int qblk = 0; qblk < QBLK; ++qblk) {
              if (qblk >= s_nqb) break;
              const uint32_t qb = qa + qblk * Q_BYTES;
              const uint32_t d = tmem + (uint32_t)(((s_g & 1) * QBLK + qblk) * BN);
#pragma unroll
              for (int kk = 0; kk < D / 16; ++kk) {
                const uint32_t off = (kk & 3) * 32;
                mma_ss(d, desc_sw128(qb + (kk >> 2) * Q_SLAB + off, 16, 1024),
                       desc_sw128(kb + (kk >> 2) * KV_SLAB + off, 16, 1024), kIdescS, kk > 0);
              }
            }
            commit(&s_ready[s_g & 1]);
            ++s_g;
            if (++s_j == s_nb) {
              s_j = 0;
              s_it += grid;
              ++s_ii;
              q_ok = false;
              s_nb = nblk_of(s_it);
              s_nqb = nqb_of(s_it);
            }
            progress = true;
          }
        }
        const int b = p_g & 1;
        if (mbar_test(&p_ready[b], (p_g >> 1) & 1)) {
          TCT(3, p_g);
          fence_after();
          const uint32_t vb = kva + (p_g % ST) * STAGE + K_BYTES;
#pragma unroll
          for (int qblk = 0; qblk < QBLK; ++qblk)
#pragma unroll
            for (int kk = 0; kk < BN / 16; ++kk)
              if (qblk < p_nqb)
              mma_ts(tmem + O_COL + qblk * D, tmem + (uint32_t)((b * QBLK + qblk) * BN + kk * 8),
                     desc_sw128(vb + kk * 2048, KV_SLAB, 1024), kIdescO, (p_j > 0 || kk > 0) ? 1u : 0u);
          commit(&pv_done[b]);
          commit(&kv_empty[p_g % ST]);
          ++p_g;
          if (++p_j == p_nb) {
            p_j = 0;
            p_it += grid;
            p_nb = nblk_of(p_it);
            p_nqb = nqb_of(p_it);
          }
          progress = true;
        }
        if (!progress) __nanosleep(20);
      }
    }
  } else if (warp < 4 * QBLK) {
    // ---------------------------------------------------------- softmax
    const int qblk = warp >> 2;                      // this warp's q-block
    const int t = threadIdx.x & (M - 1);             // MMA row / TMEM lane within the q-block
    const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    const uint32_t s_col = (uint32_t)(qblk * BN), o_col = O_COL + (uint32_t)(qblk * D);
    const int qi = qblk * (M / GRP) + t / GRP, hj = t % GRP;
    griddep_wait();                                  // q rows come from the preceding kernel
    // Q row t of this q-block of item `it` -> swizzled K-major A tile (cp.async,
    // completion counted on q_ready); the previous item's MMAs are all done.
    auto load_q = [&](int it) {
      const int32_t* rec = items + (int64_t)it * TIM_EXT_FIELDS;
      const bool ok = qi < rec[3];
      const __nv_bfloat16* src = q + ((int64_t)(rec[0] + (ok ? qi : 0)) * hq + rec[5] * GRP + hj) * D;
      uint8_t* dq = sQ + qblk * Q_BYTES;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        uint8_t* dst = dq + (c >> 3) * Q_SLAB + swz(t, c & 7);
        if (ok) cp_async16(dst, src + c * 8);
        else *reinterpret_cast<uint4*>(dst) = make_uint4(0u, 0u, 0u, 0u);
      }
      if (!ok) fence_proxy_async();
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(q_ready)) : "memory");
    };
    int gb = 0, ii = 0;
    for (int it = cta; it < n_items; it += grid, ++ii) {
      const int32_t* rec = items + (int64_t)it * TIM_EXT_FIELDS;
      const int row0 = rec[0], kv_len = rec[2], nq = rec[3], head = rec[5];
      const int nblk = (kv_len + BN - 1) / BN;
      const bool valid = qi < nq;
      const int lim = kv_len - nq + qi;              // last key this query sees (model.py:139-140)
      const int64_t qoff = ((int64_t)(row0 + qi) * hq + head * GRP + hj) * D;
      load_q(it);

      if (qblk * (M / GRP) >= nq) {
        // this q-block holds no query of the item: no MMA was issued for it,
        // its warps only keep the barrier phases (arrive once S_j exists, so
        // the arrival cannot count toward block j-2's phase)
        for (int j = 0; j < nblk; ++j, ++gb) {
          mbar_wait(&s_ready[gb & 1], (gb >> 1) & 1);
          mbar_arrive(&p_ready[gb & 1]);
        }
        mbar_wait(&pv_done[(gb - 1) & 1], ((gb - 1) >> 1) & 1);   // item done before the next Q
        continue;
      }
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < nblk; ++j, ++gb) {
        const int b = gb & 1;
        mbar_wait(&s_ready[b], (gb >> 1) & 1);
        if (threadIdx.x == 0) TCT(4, gb);
        fence_after();
        float s[64];
        {
          float a0[32], a1[32];
          tld32(lane_base + (uint32_t)(b * QBLK * BN) + s_col, a0);
          tld32(lane_base + (uint32_t)(b * QBLK * BN) + s_col + 32, a1);
          tld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            s[i] = a0[i];
            s[32 + i] = a1[i];
          }
        }
        // causal / length mask: keys k0 + i with i > vis are invisible to this row
        const int vis = (lim < kv_len - 1 ? lim : kv_len - 1) - j * BN;
        if (!__all_sync(0xffffffffu, vis >= BN - 1)) {
#pragma unroll
          for (int i = 0; i < 64; ++i) s[i] = i <= vis ? s[i] : -INFINITY;
        }
        float mq[4] = {s[0], s[1], s[2], s[3]};
#pragma unroll
        for (int i = 4; i < 64; i += 4) {
          mq[0] = fmaxf(mq[0], s[i]);
          mq[1] = fmaxf(mq[1], s[i + 1]);
          mq[2] = fmaxf(mq[2], s[i + 2]);
          mq[3] = fmaxf(mq[3], s[i + 3]);
        }
        const float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])) * scale_log2;  // scale > 0
        float m_use = m_run, corr = 1.f;
        if (mx > m_run + kRescaleLog2 || m_run == -INFINITY) {
          m_use = fmaxf(m_run, mx);
          corr = m_run == -INFINITY ? 0.f : fast_exp2(m_run - m_use);
        }
        const float msub = m_use == -INFINITY ? 0.f : m_use;
        float sq[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t pk[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float p0 = ex2f(fmaf(s[2 * i], scale_log2, -msub));
          const float p1 = ex2f(fmaf(s[2 * i + 1], scale_log2, -msub));
          sq[i & 3] += p0 + p1;
          pk[i] = pack_bf16(p0, p1);
        }
        const float sum = (sq[0] + sq[1]) + (sq[2] + sq[3]);
        l_run = l_run * corr + sum;
        m_run = m_use;
        // observe PV_{g-2} (same barrier as this block's PV; long complete) --
        // P_{g-2} lived in this S buffer and its PV ran before S_g overwrote it
        // (the tensor pipe runs in issue order); O may be rescaled only once
        // PV_{g-1} is done
        if (gb >= 2 && j >= 2) mbar_wait(&pv_done[b], ((gb - 2) >> 1) & 1);
        if (j > 0 && __any_sync(0xffffffffu, corr != 1.f)) {
          mbar_wait(&pv_done[b ^ 1], ((gb - 1) >> 1) & 1);
          fence_after();
#pragma unroll
          for (int cblk = 0; cblk < D / 32; ++cblk) {
            float o[32];
            tld32(lane_base + o_col + cblk * 32, o);
            tld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] *= corr;
            tst32(lane_base + o_col + cblk * 32, o);
          }
          tst_wait();
        }
        // P (bf16 pairs) over the first 32 columns of this block's S buffer:
        // the TMEM A operand of its PV MMA
        {
          float pf[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) pf[i] = __uint_as_float(pk[i]);
          tst32(lane_base + (uint32_t)(b * QBLK * BN) + s_col, pf);
        }
        tst_wait();
        fence_before();
        mbar_arrive(&p_ready[b]);
        if (threadIdx.x == 0) TCT(5, gb);
      }
      // epilogue: O / l of this row -> bf16 -> out.  Observe the last two PV
      // phases (one per pv_done barrier): every phase of the ring is waited on
      // by someone (the loop above waited the phases of blocks j-2).
      const int gl = gb - 1;
      if (nblk >= 2) mbar_wait(&pv_done[(gl - 1) & 1], ((gl - 1) >> 1) & 1);
      mbar_wait(&pv_done[gl & 1], (gl >> 1) & 1);
      fence_after();
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      __nv_bfloat16* orow = out + qoff;
#pragma unroll
      for (int cblk = 0; cblk < D / 32; ++cblk) {
        float o[32];
        tld32(lane_base + o_col + cblk * 32, o);
        tld_wait();
        if (valid) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint4 v;
            v.x = pack_bf16(o[8 * c] * inv, o[8 * c + 1] * inv);
            v.y = pack_bf16(o[8 * c + 2] * inv, o[8 * c + 3] * inv);
            v.z = pack_bf16(o[8 * c + 4] * inv, o[8 * c + 5] * inv);
            v.w = pack_bf16(o[8 * c + 6] * inv, o[8 * c + 7] * inv);
            *reinterpret_cast<uint4*>(orow + cblk * 32 + c * 8) = v;
          }
        }
      }
      fence_before();
    }
  }
  fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS)
                 : "memory");
  }
}

}  // namespace tim
