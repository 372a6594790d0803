// K4 (subtask prune compaction), K5 (LIFO page allocator) and row staging.
//
// Device-authoritative paging: the free stack, every request's block table and
// its aligned `live` list (logical index per table slot) live in HBM.  The host
// plans one engine step as counts only (it never needs page ids) and the
// kernels below materialise the ids with the exact reference interleaving:
//   paging.py:40      free list initialised [cap-1 .. 0]  -> first pops 0,1,2,...
//   paging.py:57      alloc pops from the top, one id per token, in order
//   paging.py:62-67   free appends ids in the given (table) order
//   pruning.py:130    the freed ids are table[suffix_start:]
//   scheduler.py:274-316 ops are sequenced admissions -> advances in submission order
#include "common.cuh"

namespace tim {

__global__ void pool_init_kernel(int32_t* free_stack, int32_t* owner, int32_t capacity) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < capacity; i += gridDim.x * blockDim.x) {
    free_stack[i] = capacity - 1 - i;  // stack[0] is the bottom; top = stack[sp-1] = 0
    owner[i] = -1;
  }
}

// One CTA of 1024 threads.  Ops of a phase are independent (the host starts a
// new phase whenever the op kind changes), so warps take ops round-robin and
// lanes stride over an op's pages; phases are separated by __syncthreads().
__global__ void __launch_bounds__(1024) page_ops_kernel(const int32_t* step, int32_t* free_stack,
                                                        int32_t* owner, int32_t capacity,
                                                        int32_t* tables, int64_t tstride,
                                                        int32_t* err) {
  const tim_step_header& h = *reinterpret_cast<const tim_step_header*>(step);
  const int32_t* ops = step + h.off_ops;
  const int32_t* phases = step + h.off_phases;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int p = 0; p < h.n_phases; ++p) {
    const int o0 = phases[p], o1 = phases[p + 1];
    for (int o = o0 + warp; o < o1; o += nwarps) {
      const int32_t* op = ops + (int64_t)o * TIM_OP_FIELDS;
      const int32_t kind = op[0], slot = op[1], toff = op[2], count = op[3], sp = op[4];
      const int32_t who = op[5];
      int32_t* trow = tables + (int64_t)slot * tstride + toff;
      if (kind == TIM_OP_ALLOC) {
        if (sp - count < 0) {
          if (lane == 0) raise_error(err, TIM_OUT_OF_PAGES, count);
          continue;
        }
        for (int j = lane; j < count; j += 32) {
          const int32_t page = free_stack[sp - 1 - j];
          if (page < 0 || page >= capacity || atomicExch(&owner[page], who) != -1)
            raise_error(err, TIM_DOUBLE_FREE, page);
          trow[j] = page;
        }
      } else {
        if (sp + count > capacity) {
          if (lane == 0) raise_error(err, TIM_DOUBLE_FREE, -1);
          continue;
        }
        for (int j = lane; j < count; j += 32) {
          const int32_t page = trow[j];
          bool ok = page >= 0 && page < capacity;
          if (ok) {
            if (who == -2) ok = atomicExch(&owner[page], -1) != -1;
            else ok = atomicCAS(&owner[page], who, -1) == who;
          }
          if (!ok) raise_error(err, TIM_DOUBLE_FREE, page);
          free_stack[sp + j] = page;
        }
      }
    }
    __syncthreads();
  }
}

// Block-wide exclusive scan of 0/1 flags (blockDim.x == 256).
__device__ __forceinline__ int block_excl_scan(int flag, int* warp_tot, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned ballot = __ballot_sync(0xffffffffu, flag);
  const int in_warp = __popc(ballot & ((1u << lane) - 1u));
  if (lane == 0) warp_tot[warp] = __popc(ballot);
  __syncthreads();
  int base = 0, tot = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
    const int v = warp_tot[w];
    base += (w < warp) ? v : 0;
    tot += v;
  }
  total = tot;
  return base + in_warp;
}

// K4: one CTA per prune job (pruning.py:102-133 restated over device arrays).
__global__ void __launch_bounds__(256) prune_compact_kernel(const int32_t* step, int32_t* live,
                                                            int64_t lstride, const int32_t* logical,
                                                            int64_t gstride, int32_t* row_tokens,
                                                            int32_t* err) {
  const tim_step_header& h = *reinterpret_cast<const tim_step_header*>(step);
  if ((int)blockIdx.x >= h.n_jobs) return;
  const int32_t* job = step + h.off_jobs + (int64_t)blockIdx.x * TIM_JOB_FIELDS;
  const int32_t slot = job[0], old_len = job[1], s = job[2], reencode_from = job[3];
  const int32_t span_off = job[4], n_spans = job[5], out_row = job[6], expect_keep = job[7];
  const int32_t* spans = step + h.off_spans + span_off * 2;
  int32_t* lrow = live + (int64_t)slot * lstride;
  const int32_t* grow = logical + (int64_t)slot * gstride;

  __shared__ int32_t sspan[2 * 64];
  __shared__ int warp_tot[8];
  const int ns = n_spans < 64 ? n_spans : 64;
  for (int i = threadIdx.x; i < 2 * ns; i += blockDim.x) sspan[i] = spans[i];
  if (threadIdx.x == 0) {
    // suffix_start = first live index >= reencode_from (pruning.py:126-128)
    const bool lo_ok = (s == 0) || (lrow[s - 1] < reencode_from);
    const bool hi_ok = (s == old_len) || (lrow[s] >= reencode_from);
    if (!lo_ok || !hi_ok || n_spans > 64) raise_error(err, TIM_SPAN_OUT_OF_RANGE, slot);
  }
  __syncthreads();

  int kept = 0;
  for (int c0 = s; c0 < old_len; c0 += blockDim.x) {
    const int idx = c0 + threadIdx.x;
    int val = 0, keep = 0;
    if (idx < old_len) {
      val = lrow[idx];
      keep = 1;
      for (int k = 0; k < ns; ++k)
        if (val >= sspan[2 * k] && val < sspan[2 * k + 1]) keep = 0;
    }
    int total;
    const int rank = block_excl_scan(keep, warp_tot, total);
    __syncthreads();  // every read of this chunk happened before any in-place write
    if (keep) {
      lrow[s + kept + rank] = val;
      if (out_row >= 0) row_tokens[out_row + kept + rank] = grow[val];
    }
    kept += total;
    __syncthreads();
  }
  if (threadIdx.x == 0 && kept != expect_keep) raise_error(err, TIM_SPAN_OUT_OF_RANGE, slot);
}

__global__ void stage_new_kernel(const int32_t* step, int32_t* live, int64_t lstride,
                                 int32_t* logical, int64_t gstride, int32_t* row_tokens) {
  const tim_step_header& h = *reinterpret_cast<const tim_step_header*>(step);
  const int32_t* nw = step + h.off_new;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < h.n_new; i += gridDim.x * blockDim.x) {
    const int32_t* r = nw + (int64_t)i * TIM_NEW_FIELDS;
    const int32_t slot = r[0], lidx = r[1], tok = r[2], row = r[3], live_idx = r[4];
    if (row == -2) continue;                   // counted by the step report only
    logical[(int64_t)slot * gstride + lidx] = tok;
    if (row >= 0) {
      live[(int64_t)slot * lstride + live_idx] = lidx;
      row_tokens[row] = tok;
    }
  }
}

__global__ void stage_rows_kernel(const int32_t* step, const int32_t* tables, int64_t tstride,
                                  int32_t* row_tokens, int32_t* row_pages, int32_t* row_pos) {
  const tim_step_header& h = *reinterpret_cast<const tim_step_header*>(step);
  const int32_t* segs = step + h.off_segs;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < h.n_rows_pad; r += gridDim.x * blockDim.x) {
    if (r >= h.n_rows) {
      row_pages[r] = -1;
      row_pos[r] = 0;
      row_tokens[r] = 0;
      continue;
    }
    // segments are sorted by row_off: binary search the owner of row r
    int lo = 0, hi = h.n_segs - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (segs[mid * TIM_SEG_FIELDS + 3] <= r) lo = mid; else hi = mid - 1;
    }
    const int32_t* sg = segs + lo * TIM_SEG_FIELDS;
    const int32_t slot = sg[0], m = sg[1], row_off = sg[3];
    const int32_t i = r - row_off;
    row_pages[r] = tables[(int64_t)slot * tstride + m + i];
    row_pos[r] = m + i;
  }
}


// StepReport / RequestMetrics from device counters (scheduler.py:320-335,
// 513-519; pruning.py:36-58).  Runs after the step's page ops and row staging:
// replays the op list against the device's own free-stack pointer (acct[0]) --
// an op whose host-planned sp_before disagrees raises TIM_DOUBLE_FREE -- keeps
// every slot's table length and high-water mark (max_cache, taken at each
// ALLOC as _touch_memory does after each forward), and counts the step's
// first-encoded rows (`new` records staged as rows): decoded tokens per slot
// and flops units sum(position + 1) (scheduler.py:374-377).  The record lands
// in a device ring, so reading metrics never synchronises the step.
constexpr int kAcctOps = 1024;   // ops staged in shared memory (a longer list runs serially)

__global__ void __launch_bounds__(256) step_account_kernel(const int32_t* step, int32_t* acct, int32_t* slot_acct,
                                                           int32_t n_slots, int32_t* reports, int32_t ring_cap,
                                                           int32_t* err) {
  const tim_step_header& h = *reinterpret_cast<const tim_step_header*>(step);
  if (slot_acct == nullptr) n_slots = 0;
  int32_t* slot_len = slot_acct;
  int32_t* slot_hw = slot_acct + n_slots;
  __shared__ unsigned long long flops;
  __shared__ int32_t sop[kAcctOps][4];       // kind, slot, table_off, count
  __shared__ int32_t sp_end;
  extern __shared__ int32_t sdec[];
  const int n_ops = h.n_ops;
  const int32_t* ops = step + h.off_ops;
  for (int i = threadIdx.x; i < n_slots; i += blockDim.x) sdec[i] = 0;
  if (threadIdx.x == 0) flops = 0ull;
  const bool staged = n_ops <= kAcctOps;
  if (staged) {
    for (int o = threadIdx.x; o < n_ops; o += blockDim.x) {
      const int32_t* op = ops + (int64_t)o * TIM_OP_FIELDS;
      sop[o][0] = op[0];
      sop[o][1] = op[1];
      sop[o][2] = op[2];
      sop[o][3] = op[3];
    }
  }
  __syncthreads();
  const int32_t* nw = step + h.off_new;
  for (int i = threadIdx.x; i < h.n_new; i += blockDim.x) {
    const int32_t* r = nw + (int64_t)i * TIM_NEW_FIELDS;
    if (r[3] == -1) continue;                    // logged, not encoded this step
    // row -2: first-encoded by the reference's forward, not staged here (its
    // request ended this step): flops units only
    if (r[3] >= 0 && r[0] < n_slots) atomicAdd(&sdec[r[0]], 1);
    atomicAdd(&flops, (unsigned long long)(r[4] + 1));
  }
  if (staged) {
    // free-stack pointer: warp 0 scans the ops' deltas; every host-planned
    // sp_before must equal the device's running pointer
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      int32_t sp = acct[0];
      for (int o0 = 0; o0 < n_ops; o0 += 32) {
        const int o = o0 + lane;
        int32_t d = 0;
        if (o < n_ops) d = sop[o][0] == TIM_OP_ALLOC ? -sop[o][3] : sop[o][3];
        int32_t inc = d;
#pragma unroll
        for (int k = 1; k < 32; k <<= 1) {
          const int32_t v = __shfl_up_sync(0xffffffffu, inc, k);
          if (lane >= k) inc += v;
        }
        if (o < n_ops && ops[(int64_t)o * TIM_OP_FIELDS + 4] != sp + inc - d) raise_error(err, TIM_DOUBLE_FREE, -3);
        sp += __shfl_sync(0xffffffffu, inc, 31);
      }
      if (lane == 0) sp_end = sp;
    }
    // per slot: its ops in order (table length; high-water mark at each ALLOC,
    // reset when a table restarts at index 0 for a new request)
    for (int sl = threadIdx.x; sl < n_slots; sl += blockDim.x) {
      int32_t len = slot_len[sl], hw = slot_hw[sl];
      for (int o = 0; o < n_ops; ++o) {
        if (sop[o][1] != sl) continue;
        if (sop[o][0] == TIM_OP_ALLOC) {
          if (sop[o][2] == 0) hw = 0;
          len = sop[o][2] + sop[o][3];
          hw = len > hw ? len : hw;
        } else {
          len = sop[o][2];
        }
      }
      slot_len[sl] = len;
      slot_hw[sl] = hw;
    }
  } else if (threadIdx.x == 0) {
    int32_t sp = acct[0];
    for (int o = 0; o < n_ops; ++o) {
      const int32_t* op = ops + (int64_t)o * TIM_OP_FIELDS;
      const int32_t kind = op[0], slot = op[1], toff = op[2], count = op[3], sp_before = op[4];
      if (sp_before != sp) raise_error(err, TIM_DOUBLE_FREE, -3);
      sp += kind == TIM_OP_ALLOC ? -count : count;
      if (slot < n_slots) {
        if (kind == TIM_OP_ALLOC) {
          if (toff == 0) slot_hw[slot] = 0;
          slot_len[slot] = toff + count;
          if (toff + count > slot_hw[slot]) slot_hw[slot] = toff + count;
        } else {
          slot_len[slot] = toff;
        }
      }
    }
    sp_end = sp;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    acct[0] = sp_end;
    acct[1] += 1;
  }
  __syncthreads();
  if (reports == nullptr || ring_cap <= 0) return;
  const int rec_len = 4 + 3 * n_slots;
  int32_t* rec = reports + (int64_t)((acct[1] - 1) % ring_cap) * rec_len;
  if (threadIdx.x == 0) {
    rec[0] = h.serial;
    rec[1] = sp_end;
    rec[2] = (int32_t)(flops & 0xffffffffull);
    rec[3] = (int32_t)(flops >> 32);
  }
  for (int i = threadIdx.x; i < n_slots; i += blockDim.x) {
    rec[4 + 3 * i] = slot_len[i];
    rec[5 + 3 * i] = sdec[i];
    rec[6 + 3 * i] = slot_hw[i];
  }
}
}  // namespace tim

using namespace tim;

extern "C" int32_t tim_pool_init(int32_t* free_stack, int32_t* owner, int32_t capacity, void* stream) {
  if (capacity < 1) { set_last_error("capacity must be >= 1"); return TIM_BAD_ARGUMENT; }
  const int threads = 256;
  const int blocks = (capacity + threads - 1) / threads < 1024 ? (capacity + threads - 1) / threads : 1024;
  pool_init_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(free_stack, owner, capacity);
  return check_launch("pool_init");
}

extern "C" int32_t tim_page_ops(const int32_t* step, int32_t* free_stack, int32_t* owner,
                                int32_t capacity, int32_t* block_tables, int64_t table_stride,
                                int32_t* err, void* stream) {
  prefer_shared(page_ops_kernel);
  page_ops_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(step, free_stack, owner, capacity,
                                                         block_tables, table_stride, err);
  return check_launch("page_ops");
}

extern "C" int32_t tim_prune_compact(const int32_t* step, int32_t max_jobs, int32_t* live,
                                     int64_t live_stride, const int32_t* logical,
                                     int64_t logical_stride, int32_t* row_tokens, int32_t* err,
                                     void* stream) {
  if (max_jobs <= 0) return TIM_OK;
  prefer_shared(prune_compact_kernel);
  prune_compact_kernel<<<max_jobs, 256, 0, (cudaStream_t)stream>>>(step, live, live_stride, logical,
                                                                   logical_stride, row_tokens, err);
  return check_launch("prune_compact");
}

extern "C" int32_t tim_stage_rows(const int32_t* step, const int32_t* block_tables,
                                  int64_t table_stride, int32_t* live, int64_t live_stride,
                                  int32_t* logical, int64_t logical_stride, int32_t* row_tokens,
                                  int32_t* row_pages, int32_t* row_pos, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  prefer_shared(stage_new_kernel);
  stage_new_kernel<<<16, 256, 0, st>>>(step, live, live_stride, logical, logical_stride, row_tokens);
  int32_t rc = check_launch("stage_new");
  if (rc) return rc;
  prefer_shared(stage_rows_kernel);
  stage_rows_kernel<<<16, 256, 0, st>>>(step, block_tables, table_stride, row_tokens, row_pages, row_pos);
  return check_launch("stage_rows");
}

extern "C" int32_t tim_step_account(const int32_t* step, int32_t* acct, int32_t* slot_acct, int32_t n_slots,
                                    int32_t* reports, int32_t ring_cap, int32_t* err, void* stream) {
  if (n_slots < 0 || n_slots > 8192) { set_last_error("n_slots out of range"); return TIM_BAD_ARGUMENT; }
  prefer_shared(step_account_kernel);
  step_account_kernel<<<1, 256, (size_t)(n_slots > 0 ? n_slots : 1) * sizeof(int32_t), (cudaStream_t)stream>>>(
      step, acct, slot_acct, n_slots, reports, ring_cap, err);
  return check_launch("step_account");
}
