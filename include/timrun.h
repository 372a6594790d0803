/*
 * timrun.h — C ABI of libtimrun.so, the B200 (sm_100a) working-memory decode path.
 *
 * This is the drop-in boundary for the reference runtime `threadrun`
 * (/root/reference/pkg/src/threadrun).  The reference's plugin interface for
 * this path is the duck-typed model-backend protocol consumed by `Engine`
 * (scheduler.py:198-205,350,372; model.py:115-183) plus the page pool and
 * prune entry points it drives (paging.py:27-107, pruning.py:102-133).  Every
 * function below replaces one piece of that interface; the citation on each
 * names the reference code it replaces.  All pointers are device pointers
 * unless noted, sizes are plain integers, `stream` is a cudaStream_t passed as
 * void*.  No function synchronises the host except tim_read_error().
 *
 * Step descriptor.  One engine step is described by a single int32 buffer
 * (`step`, device-resident, uploaded with one H2D copy) that starts with a
 * tim_step_header; record arrays follow at the header's offsets.  All kernels
 * of a step read the same buffer, so the host never re-uploads metadata and
 * the whole step is CUDA-graph capturable.
 */
#ifndef TIMRUN_H
#define TIMRUN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes.  Each maps onto the reference exception named beside it. */
enum {
  TIM_OK = 0,
  TIM_OUT_OF_PAGES = 1,       /* paging.py:14-18   OutOfPages(needed, available) */
  TIM_DOUBLE_FREE = 2,        /* paging.py:21-24   DoubleFree(page_id)           */
  TIM_POSITION_OVERFLOW = 3,  /* model.py:24-28    PositionOverflow(pos, limit)  */
  TIM_SPAN_OUT_OF_RANGE = 4,  /* pruning.py:25-26  SpanOutOfRange (desync)       */
  TIM_BAD_ARGUMENT = 5,       /* ValueError                                      */
  TIM_CUDA_ERROR = 6,
  TIM_UNSUPPORTED = 7,
  TIM_REJECTED = 8            /* tracker.py:56-65  Rejected (token not admitted) */
};

enum { TIM_DTYPE_F32 = 0, TIM_DTYPE_BF16 = 1 };

/* Page-op kinds (records in the step descriptor). */
enum {
  TIM_OP_ALLOC = 0,  /* pop `count` ids off the LIFO free stack (paging.py:52-60) into table[slot][off..] */
  TIM_OP_FREE = 1    /* push table[slot][off..off+count) in table order (paging.py:62-67)          */
};

/* Header of the per-step descriptor.  Offsets are int32 element offsets into
 * the same buffer.  Record layouts (int32 fields):
 *   new   : {slot, logical_idx, token, row, live_idx}          host-known tokens
 *           (row -1: logged, not encoded; -2: counted by tim_step_account only)
 *   last  : rows whose logits are produced, then last_mask: one mask id per
 *           `last` entry for tim_masked_argmax (-1: unmasked)
 *   seg   : {slot, m, n, row_off}                               one encode segment
 *   dec   : {row, slot, kv_len, nq, m, group} + dec_prefix[n_dec+1]
 *                                   decode tiles (1 query x all kv heads; m = first fresh key)
 *   ext   : {row, slot, kv_len, nq, m, group} + ext_prefix[n_ext+1]
 *                                   multi-token tiles (queries x one kv-head group)
 *   job   : {slot, old_len, suffix_start, reencode_from,
 *            span_off, n_spans, out_row, expect_keep}           prune compaction jobs
 *   spans : {start, end}                                        coalesced evict spans
 *   op    : {kind, slot, table_off, count, sp_before, owner}    page ops (owner -2: any)
 *   phase : n_phases+1 op offsets (ops within a phase are independent)
 *   last  : {row}                                               rows whose logits are produced
 */
typedef struct {
  int32_t n_rows, n_rows_pad;
  int32_t n_new, n_segs, n_dec, n_ext, n_jobs, n_ops, n_phases, n_last;
  int32_t dec_total;
  int32_t off_new, off_segs, off_dec, off_dec_prefix, off_ext, off_jobs, off_spans;
  int32_t off_ops, off_phases, off_last;
  int32_t ext_total, off_ext_prefix;
  int32_t split_dec_ctas, split_ext_ctas;  /* mode-2 attention: CTAs on dec tiles / ext items */
  int32_t serial;                          /* step serial (!= 0) matching tim_attn_plan's record */
  int32_t reserved[6];
} tim_step_header;  /* 32 int32 */

#define TIM_NEW_FIELDS 5
#define TIM_SEG_FIELDS 4
#define TIM_DEC_FIELDS 6
#define TIM_EXT_FIELDS 6
#define TIM_JOB_FIELDS 8
#define TIM_OP_FIELDS 6

/* ---------------------------------------------------------------- utility */
int32_t tim_abi_version(void);
const char* tim_last_error(void);               /* host string of the last failure */
int32_t tim_sm_count(void);                     /* SMs of the current device */
/* Blocking read of the device error word (err[0] code, err[1] detail); clears it. */
int32_t tim_read_error(int32_t* err_dev, int32_t* code_out, int32_t* detail_out, void* stream);

/* ------------------------------------------------------ pool / allocator (K5) */
/* Free stack initialised to [cap-1, ..., 0] so pops return 0,1,2,... (paging.py:40),
 * owner[] = -1 (paging.py:41). */
int32_t tim_pool_init(int32_t* free_stack, int32_t* owner, int32_t capacity, void* stream);

/* K5 + K4-free: run the step's phased page ops against the device LIFO free stack.
 * ALLOC pops ids top-first (paging.py:57), FREE pushes table entries in table
 * order (paging.py:62-67, pruning.py:130 truncate_from, scheduler.py:398,522,539).
 * Owner checks raise TIM_DOUBLE_FREE in err[]; stack under/overflow raises
 * TIM_OUT_OF_PAGES.  One CTA; phases are separated by block barriers. */
int32_t tim_page_ops(const int32_t* step, int32_t* free_stack, int32_t* owner, int32_t capacity,
                     int32_t* block_tables, int64_t table_stride, int32_t* err, void* stream);

/* StepReport / RequestMetrics from device counters (scheduler.py:320-335,513-519;
 * pruning.py:36-58).  After a step's page ops and row staging: replay the op
 * list against the pool's device free-stack pointer acct[0] (a host-planned
 * sp_before that disagrees raises TIM_DOUBLE_FREE), count steps in acct[1]
 * (acct starts as {capacity, 0}); with slot_acct ([2][n_slots], zeroed), keep
 * every slot's table length and high-water mark (max_cache, taken at each
 * ALLOC as _touch_memory does after each forward), count the step's
 * first-encoded rows per slot and their flops units sum(position+1)
 * (scheduler.py:374-377), and write the record {serial, pages_free, flops_lo,
 * flops_hi, (len, decoded, max_cache) x n_slots} to ring entry
 * (acct[1] - 1) % ring_cap of `reports` (NULL: no record). */
int32_t tim_step_account(const int32_t* step, int32_t* acct, int32_t* slot_acct, int32_t n_slots,
                         int32_t* reports, int32_t ring_cap, int32_t* err, void* stream);

/* -------------------------------------------------------- subtask prune (K4) */
/* For each prune job: verify suffix_start against live[] (the first index with
 * live >= reencode_from, pruning.py:126-128), mark retained entries of
 * live[s:old_len) not covered by the coalesced evict spans (pruning.py:131),
 * compact them in place (new_live[s:]), and gather their token ids from the
 * device logical stream into the step's row_tokens at out_row
 * (pruning.py:132 suffix_tokens; scheduler.py:403-405).  Count mismatches
 * against the host plan raise TIM_SPAN_OUT_OF_RANGE. */
int32_t tim_prune_compact(const int32_t* step, int32_t max_jobs, int32_t* live, int64_t live_stride,
                          const int32_t* logical, int64_t logical_stride, int32_t* row_tokens,
                          int32_t* err, void* stream);

/* Stage the step's rows: write host-known new tokens into the device logical
 * stream, live[] and row_tokens; then for every segment row compute its page
 * (table[slot][m+i], appended by the ALLOC ops) and position m+i (position
 * recycling: scheduler.py:366-372, model.py:174-179).  Rows past n_rows up to
 * n_rows_pad get page -1 (no KV write). */
int32_t tim_stage_rows(const int32_t* step, const int32_t* block_tables, int64_t table_stride,
                       int32_t* live, int64_t live_stride, int32_t* logical, int64_t logical_stride,
                       int32_t* row_tokens, int32_t* row_pages, int32_t* row_pos, void* stream);

/* ------------------------------------------------------- model-side kernels */
/* h[r,:] = emb[row_tokens[r], :]  (model.py:138) */
int32_t tim_embed(const int32_t* row_tokens, int32_t n_rows, const void* emb, int32_t dm,
                  void* h, int32_t dtype, void* stream);
/* y = x / sqrt(mean(x^2) + eps) (model.py:69-70); fp32 math, rows of length dm. */
int32_t tim_rmsnorm(const void* x, int64_t x_stride, void* y, int64_t y_stride, int32_t n_rows,
                    int32_t dm, float eps, int32_t dtype, void* stream);
/* in-place x = x / (1 + exp(-x)) (model.py:73-74) */
int32_t tim_silu(void* x, int64_t n, int32_t dtype, void* stream);

/* K3: rotate-half RoPE (model.py:118-125) of q and k from the fused qkv GEMM
 * output [rows, (hq + 2 hkv) * D], store roped K and V into the page of each
 * row for this layer (model.py:147-148), write roped q to q_out.  When `h` is
 * non-null the row's weightless RMSNorm (model.py:69-70) is applied here as a
 * per-row scale 1/sqrt(mean(h^2)+eps): the GEMM ran on the raw residual h,
 * and rms(h) @ W == (h @ W) * scale.  cos/sin tables are [position_limit,
 * D/2] fp32, built on the host exactly as the reference (fp32 angle
 * pos*inv_freq, model.py:104-105,121). */
int32_t tim_rope_kv_store(const void* qkv, const void* h, int32_t dm, float eps, int32_t n_rows,
                          const int32_t* row_pos, const int32_t* row_pages, const float* cos_tab,
                          const float* sin_tab, int32_t hq, int32_t hkv, int32_t head_dim,
                          void* q_out, void* k_layer, void* v_layer, int32_t dtype, void* stream);
/* u[r,:] = silu(u[r,:] * 1/sqrt(mean(h[r,:]^2)+eps)) in place: the MLP input
 * RMSNorm folded behind the W1 GEMM (model.py:161). */
int32_t tim_silu_rms(void* u, int32_t n_rows, int32_t width, const void* h, int32_t dm, float eps,
                     int32_t dtype, void* stream);

/* K1+K2+K6: paged GQA attention over retained pages only (model.py:149-159),
 * replacing the per-request attention loop of TinyTransformer._forward
 * (model.py:142-161) called from Engine._advance (scheduler.py:372).  Work
 * items are query tiles {row, slot, kv_len, nq, m, group}: nq consecutive
 * query rows of one request; query i of a tile sees keys [0, kv_len - nq + i]
 * (prefix fully visible, causal inside the new block); keys >= m were written
 * by this step.
 *   mode 0: the step's decode tiles (`dec`: tile_q queries x all kv heads,
 *           whole page rows), split-K over `n_ctas` persistent CTAs (stream-K);
 *           tiles spanning several CTAs are merged in-kernel (log-sum-exp).
 *   mode 1: the multi-token items (`ext`: tim_extend_queries_per_item queries
 *           x one of tim_extend_head_groups kv-head groups); on the tcgen05
 *           shape (D = 128, Hq = 4 Hkv) one item = 128 MMA rows in TMEM.
 *   mode 2: both lists in ONE launch, CTAs split per the descriptor's
 *           split_dec_ctas / split_ext_ctas (two launches where no tcgen05
 *           kernel exists for the shape).
 * Launched with programmatic dependent launch; older pages stream before the
 * preceding RoPE+store kernel finishes.
 * ws: float workspace of tim_decode_ws_floats(n_ctas, max_dec, hkv, D) floats;
 * counters: int32[max_dec * 8] zero-initialised once (self-resetting); max_dec
 * bounds the tile count. */
int64_t tim_decode_ws_floats(int32_t n_ctas, int32_t max_dec, int32_t hkv, int32_t head_dim);
int32_t tim_attn_decode(const int32_t* step, int32_t mode, const void* q, void* out,
                        const void* k_layer, const void* v_layer, const int32_t* block_tables,
                        int64_t table_stride, int32_t hq, int32_t hkv, int32_t head_dim,
                        float scale, float* ws, int32_t* counters, int32_t n_ctas, int32_t max_dec,
                        int32_t dtype, void* stream);
/* Per-step plan of the decode-tile partition (each K1 CTA's first tile and
 * the page ids of its first two stages), written into the tail of `ws` once
 * per step after the page ops (the partition is the same for every layer);
 * K1 uses it when the descriptor's serial matches, else it searches itself.
 * n_ctas / max_dec / head_dim as passed to tim_attn_decode. */
int32_t tim_attn_plan(const int32_t* step, const int32_t* block_tables, int64_t table_stride, int32_t n_ctas,
                      int32_t max_dec, int32_t head_dim, float* ws, void* stream);
/* Queries per multi-token tile and kv-head groups per query for a config. */
int32_t tim_extend_queries_per_item(int32_t hq, int32_t hkv, int32_t head_dim, int32_t dtype);
int32_t tim_extend_head_groups(int32_t hq, int32_t hkv, int32_t head_dim);

/* Diagnostics: per-CTA %globaltimer timeline of tim_attn_decode written to
 * buf[8*cta .. 8*cta+6] = {start, first stage landed, main loop end, end,
 * producer: first tile known, first page ids in hand, first stage issued};
 * pass NULL to disable. */
int32_t tim_set_trace(void* buf);
/* Diagnostics: an empty grid launched like the attention kernel (n_ctas x
 * threads, smem dynamic bytes, programmatic launch): the fixed cost that
 * CUDA-event bracketing of one launch measures. */
int32_t tim_noop(int32_t n_ctas, int32_t threads, int32_t smem, void* stream);
/* Diagnostics: per-64-key-block %globaltimer stamps of CTA 0 of the tcgen05
 * multi-token kernel, buf[8*block + {0..5}]; NULL disables. */
int32_t tim_tc_trace(void* buf);

/* Reference-precision attention (fp32, or shapes outside the tensor-core
 * kernel): every row of the step's segments attends its paged prefix plus the
 * causal new block (model.py:139-140,149-159); max_items bounds the rows. */
int32_t tim_attn_extend(const int32_t* step, int32_t max_items, const void* q, void* out,
                        const void* k_layer, const void* v_layer, const int32_t* block_tables,
                        int64_t table_stride, int32_t hq, int32_t hkv, int32_t head_dim,
                        float scale, int32_t dtype, void* stream);

/* Greedy argmax over rows of logits [n, vocab] (lowest id on ties, model.py:186-192). */
int32_t tim_argmax(const void* logits, int32_t n_rows, int32_t vocab, int32_t* out,
                   int32_t dtype, void* stream);

/* Masked greedy pick (model.py:186-192, sample(logits, mask)): row r picks the
 * highest logit among the ids set in mask row `mask_ids[r]` of the device mask
 * table `masks` ([n_masks][words] uint32, bit t of word t/32 = id t admitted),
 * lowest id on ties; mask_ids[r] < 0 = unmasked.  A row whose mask admits no
 * id < vocab writes -1 (EmptyMask, model.py:189-190). */
int32_t tim_masked_argmax(const void* logits, int32_t n_rows, int32_t vocab, const int32_t* mask_ids,
                          const uint32_t* masks, int32_t words, int32_t* out, int32_t dtype, void* stream);

/* ---------------------------------------------------------------------------
 * Grammar tracker (host memory, no CUDA): replaces threadrun's Tracker
 * (tracker.py:214-820) -- lifecycle events of the reasoning-tree document and
 * the memoised admissible-next-token masks of allowed_mask (tracker.py:319-353).
 * ------------------------------------------------------------------------- */
typedef struct tim_grammar tim_grammar;
typedef struct tim_tracker tim_tracker;

/* Event kinds (tracker.py:33-40). */
enum {
  TIM_EV_TASK_OPENED = 0,
  TIM_EV_THOUGHT_CLOSED = 1,
  TIM_EV_TOOL_PARAMS_READY = 2,
  TIM_EV_TOOL_RESULT_SLOT_OPENED = 3,
  TIM_EV_SUBTASK_LIST_OPENED = 4,
  TIM_EV_SUBTASK_LIST_CLOSED = 5,  /* a = span_start, b = span_end */
  TIM_EV_TASK_CLOSED = 6,
  TIM_EV_DONE = 7
};

/* ThreadGrammar(tools, depth_limit, tokenizer) (tracker.py:177-200): token
 * pieces as concatenated bytes + n+1 offsets; tool names likewise.
 * NULL on a bad argument. */
tim_grammar* tim_grammar_create(const uint8_t* piece_bytes, const int32_t* piece_offsets, int32_t n_pieces,
                                const uint8_t* tool_bytes, const int32_t* tool_offsets, int32_t n_tools,
                                int32_t depth_limit);
void tim_grammar_destroy(tim_grammar* g);
/* Masks created so far (ids 0..count-1, creation order) and words per mask. */
int32_t tim_grammar_mask_count(const tim_grammar* g);
int32_t tim_grammar_mask_words(const tim_grammar* g);
/* Copy out mask `mask_id` (host memory): admitted ids, the admitted ids that
 * complete the document, and the admitted count.  Any pointer may be NULL. */
int32_t tim_grammar_mask(const tim_grammar* g, int32_t mask_id, uint32_t* words, uint32_t* finish_words,
                         int32_t* count);

/* Tracker over one request's emission stream (grammar.tracker(), tracker.py:206-208). */
tim_tracker* tim_tracker_create(tim_grammar* g);
tim_tracker* tim_tracker_clone(const tim_tracker* t);
void tim_tracker_destroy(tim_tracker* t);
/* Tracker.feed (tracker.py:301-310): TIM_OK or TIM_REJECTED; *n_events events
 * of this token, read with tim_tracker_event (fields = kind, offset, depth, a, b;
 * name/params = the tool name and parameters text of tool events, valid until
 * the next feed). */
int32_t tim_tracker_feed(tim_tracker* t, int32_t token_id, int32_t* n_events);
int32_t tim_tracker_feed_many(tim_tracker* t, const int32_t* ids, int32_t n, int32_t* at);
int32_t tim_tracker_event(const tim_tracker* t, int32_t i, int32_t* fields, const char** name,
                          int32_t* name_len, const char** params, int32_t* params_len);
/* allowed_mask (tracker.py:319-335): memo id of the current state's mask. */
int32_t tim_tracker_mask(tim_tracker* t, int32_t* mask_id, int32_t* count, int32_t* can_finish);
int32_t tim_tracker_state(const tim_tracker* t, int32_t* consumed, int32_t* done, int32_t* depth,
                          int32_t* reject_byte);
const char* tim_tracker_context(const tim_tracker* t);

#ifdef __cplusplus
}
#endif
#endif /* TIMRUN_H */
