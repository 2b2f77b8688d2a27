/*
 * mla_b200.h -- C ABI of the B200-native LU hot path (libmla_b200.so).
 *
 * The reference package `mla` (arXiv 1611.06365) is pure Python + numba and has no FFI of its own;
 * its drop-in boundary is the module API in pkg/src/mla/__init__.py:6-33.  Each entry point below
 * backs exactly one of those Python callables (cited per function); the ctypes binding a maintainer
 * of the reference would add is shown in INTEGRATION.md and shipped as
 * paper_1611_06365_b200/_capi.py.
 *
 * Conventions
 *  - All matrices are column-major float64 in DEVICE memory unless the name ends in _host:
 *    element (i,j) of a view is a[i + j*ld].  Views (sub-matrices) are expressed by pointer + ld,
 *    exactly like the reference's numpy views (matrix.py:1-6).
 *  - Pivots are int32 on the device (BASELINE.json), view-local, 0-based, ipiv[k] >= k
 *    (matrix.py:74-92).  The Python layer widens to int64 (lu.py:86-89).
 *  - Every call is asynchronous on `stream` (a cudaStream_t passed as void*) unless stated.
 *  - Return value: 0 on success, <0 on failure (MLA_E_*).  Nothing throws.  A numerically singular
 *    matrix is NOT an error: it is reported through *singular (lu.py:56-59).
 *  - The caller owns all matrices; the library owns only the workspace behind mla_handle.
 *  - One handle per device, used from one host thread at a time (the reference's "collective over
 *    a team" calling convention, pool.py:3-8, collapses to a single stream-ordered call).
 */
#ifndef MLA_B200_H
#define MLA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mla_handle_s* mla_handle;

enum {
  MLA_OK = 0,
  MLA_E_INVALID = -1,   /* shape / argument error -> ValueError in the Python layer          */
  MLA_E_CUDA = -2,      /* a CUDA runtime call failed (mla_last_cuda_error gives the code)    */
  MLA_E_ABORT = -3,     /* device-side watchdog fired (protocol bug / hang avoided)           */
  MLA_E_INDEX = -4,     /* pivot index out of range -> IndexError (kernels.py:326-327)        */
  MLA_E_NOMEM = -5
};

/* Scheduling variants of lu_la (config.py:12 VARIANTS). */
enum {
  MLA_VARIANT_LU = 0,        /* no look-ahead: update then panel, whole GPU as one team        */
  MLA_VARIANT_LU_LA = 1,     /* look-ahead: panel team (sm_pf SMs) || update team              */
  MLA_VARIANT_LU_WS_STATIC = 2, /* look-ahead + join at q column-chunk boundaries              */
  MLA_VARIANT_LU_MB = 3,     /* look-ahead + worker sharing (panel SMs join the tile queue)    */
  MLA_VARIANT_LU_ET = 4      /* + early termination of the panel by the update team            */
};

/* Outcome of a factorization -- mirrors LuResult (lu.py:33-41) plus the full width schedule. */
typedef struct {
  int32_t cols_factored;
  int32_t singular;
  int32_t et_events;
  int32_t n_panels;         /* number of panels factored (prologue included)                  */
  int32_t ws_joins;         /* iterations in which panel SMs joined the update queue (WS)     */
  int32_t sm_pf_peak;       /* largest panel team used (== sm_pf unless mla_set_panel_sms_max)  */
  int32_t reserved[2];
} mla_lu_info;

/* Workspace / lifetime.  mla_create binds to `device` (cudaSetDevice) and sizes the persistent
 * grid to the device's SM count.  Synchronous. */
int mla_create(int device, mla_handle* out);
int mla_destroy(mla_handle h);
int mla_num_sms(mla_handle h);
int mla_last_cuda_error(mla_handle h);
const char* mla_version(void);

/* gemm_malleable(c, a, b, alpha, beta, flag=...)  -- kernels.py:205-234.
 * C (m x n) := alpha*C + beta*A(m x k)*B(k x n) on FP64 tensor cores.  m==0||n==0: no-op;
 * k==0: C *= alpha.  join_flag (device word, nullable) is the WS entry point of the reference:
 * `donor_ctas` CTAs of the grid stay out of the tile queue until *join_flag != 0 (polled at tile
 * granularity), then join it; with a null flag every CTA works from the start. */
int mla_gemm(mla_handle h, double* C, int64_t m, int64_t n, int64_t ldc, const double* A, int64_t lda,
             const double* B, int64_t ldb, int64_t k, double alpha, double beta,
             const uint32_t* join_flag, int donor_ctas, void* stream);

/* trsm_llu(a11, b) -- kernels.py:264-293.  B (w x c) := trilu(L)^-1 B, unit diagonal never read.  For
 * w <= 1024 the solve runs in 128-row steps through the FP64 tensor-core tile engine with explicitly inverted
 * 128 x 128 diagonal blocks (computed by a first small launch); beyond that in 32-row substitution steps. */
int mla_trsm_llu(mla_handle h, const double* L, int64_t w, int64_t ldl, double* B, int64_t c,
                 int64_t ldb, void* stream);

/* laswp(a, piv, reverse) -- kernels.py:296-332.  Interchange t <-> ipiv[t] on every column of the
 * rows x cols view, ascending (descending when reverse).  ipiv is a DEVICE int32 array of any length
 * npiv <= rows, every entry anywhere in [0, rows) (also above its own position, like the reference);
 * vectors longer than 1024 are applied in chunks of 1024 inside the call.  The whole vector is
 * range-checked on the device before anything is touched: on a bad index NOTHING is modified and the
 * (synchronous) return value is MLA_E_INDEX. */
int mla_laswp(mla_handle h, double* A, int64_t rows, int64_t cols, int64_t ld, const int32_t* ipiv,
              int64_t npiv, int reverse, void* stream);

/* Same without the synchronous read-back of the validation result (fully asynchronous): a bad index
 * still leaves the matrix untouched, it is just not reported.  Used by stream-ordered callers whose
 * pivots come straight from the panel kernel (multi-GPU path). */
int mla_laswp_async(mla_handle h, double* A, int64_t rows, int64_t cols, int64_t ld, const int32_t* ipiv,
                    int64_t npiv, int reverse, void* stream);

/* lu_blk_ll(a, b, ipiv, stop) -- lu.py:140-180 (panel factorization, left-looking, inner block
 * b_inner; b_inner >= w gives lu_unb, lu.py:97-103).  stop_flag (device word, nullable) is the ET
 * flag: polled once per completed inner block while columns remain; stop_after_polls > 0 instead
 * emulates the reference's CountingFlag fake (set from that poll on; test_lu.py:149-156).
 * team_ctas <= 0 picks a team size from m.  Synchronous (returns the info). */
int mla_panel_ll(mla_handle h, double* P, int64_t m, int64_t w, int64_t ld, int32_t* ipiv, int b_inner,
                 const uint32_t* stop_flag, int stop_after_polls, int team_ctas, mla_lu_info* info,
                 void* stream);

/* Asynchronous form for stream-ordered drivers (distributed.py): pivots stay on the device, nothing is
 * read back; the factored width / singular flag stay in the handle's device-side info record (read by
 * mla_pack_panel); singular_accum (device int32, nullable) is OR-ed with the panel's singular flag.
 * stop_flag (device word, nullable) is the ET flag of lu.py:177-179: the panel is cut after a finished
 * inner block, while columns remain, once *stop_flag == stop_tag (stop_tag == 0: once it is non-zero).
 * The panel runs in Crout order, so after a cut the leftover columns hold the interchanges and their U
 * rows (what `pend` records in lu.py:247-255, 324) -- the same contract as the persistent kernel's panels. */
int mla_panel_ll_async(mla_handle h, double* P, int64_t m, int64_t w, int64_t ld, int32_t* ipiv, int b_inner,
                       int team_ctas, int32_t* singular_accum, const uint32_t* stop_flag, uint32_t stop_tag,
                       void* stream);

/* lu_la(a, policy, pool) -- lu.py:197-334.  Whole factorization P*A = L*U in place, one persistent
 * cooperative kernel: SM partition (sm_pf panel CTAs), atomic tile queue, WS and ET by device
 * flags.  ipiv: device int32[n], global 0-based.  widths (device int32[widths_cap], nullable)
 * receives every panel's factored width in order.  info_dev (device, nullable) receives the
 * mla_lu_info; the call is asynchronous. */
int mla_getrf_la(mla_handle h, double* A, int64_t m, int64_t n, int64_t ld, int32_t* ipiv, int b_outer,
                 int b_inner, int variant, int sm_pf, int q_chunks, mla_lu_info* info_dev,
                 int32_t* widths, int widths_cap, void* stream);

/* Malleable SM split for the following mla_getrf_la* calls on this handle.  0 (default) keeps the
 * reference's behaviour: the panel team has sm_pf SMs in every iteration (the split is restored each
 * iteration, lu.py:270-273; WS only lends panel SMs to the update inside an iteration).
 * sm_pf_max > sm_pf additionally lets the panel team grow between iterations -- doubled, up to
 * sm_pf_max, after an iteration whose panel finished after the remainder update, halved (not below
 * sm_pf) after one whose panel took under a third of the iteration.  Pivots do not depend on the
 * split (factors: last-bit differences when the team size changes the panel's device block width).  Returns MLA_E_INVALID for negative values. */
int mla_set_panel_sms_max(mla_handle h, int sm_pf_max);

/* Same, reading the info back (synchronises the stream). */
int mla_getrf_la_sync(mla_handle h, double* A, int64_t m, int64_t n, int64_t ld, int32_t* ipiv,
                      int b_outer, int b_inner, int variant, int sm_pf, int q_chunks,
                      mla_lu_info* info_host, int32_t* widths_host, int widths_cap, void* stream);

/* Releases the device matrix / pivot buffers mla_getrf_la_host keeps cached in the handle. */
int mla_release_host_cache(mla_handle h);

/* End-to-end form with HOST buffers (what bench.py's `e2e` times): uploads A (m x n, ld_host),
 * factors on the device, downloads the packed factors and the pivots.  The download overlaps the
 * factorization: rows above the current panel are final (every later interchange, solve and update
 * touches lower rows only), the kernel reports that row through a mapped host word, and the finished
 * row blocks are copied out on a second stream while the kernel is still running.  The upload overlaps it as
 * well (mla_set_host_phases below).  Synchronous: the
 * calling thread polls that word (50 us sleeps) and issues the copies.  The device copy of the matrix
 * (8 * m * n bytes, e.g. 8 GiB at n = 32768) and the pivot buffer stay cached in the handle for the next
 * call of the same or a smaller size, until mla_release_host_cache or mla_destroy. */
int mla_getrf_la_host(mla_handle h, double* A_host, int64_t m, int64_t n, int64_t ld_host,
                      int32_t* ipiv_host, int b_outer, int b_inner, int variant, int sm_pf,
                      int q_chunks, mla_lu_info* info_host);

/* Windows of mla_getrf_la_host (the upload is overlapped too): the columns are uploaded in chunks and the
 * factorization runs window by window behind the upload, left-looking between windows -- window [c0, c1) waits
 * for its own chunk only, receives the interchanges / solves / updates of the columns [0, c0) factored so far
 * (catch-up), and is then factored by the persistent kernel restricted to it (look-ahead, WS and ET inside the
 * window; lu_la's own iteration structure, lu.py:243-326, from column c0 on).
 *   bounds/count: window ends in columns, ascending (rounded down to whole multiples of b_outer; the last window
 *          always ends at n); count == 0: one window (upload, then factor); count < 0 (default): windows end at
 *          n/32, n/8 and 3n/8 for n >= 8192.
 *   deep:  0: the catch-up applies one b_outer block at a time (solve + rank-b update of all rows below) -- every
 *          matrix entry then sees the same operations in the same order as in an unwindowed run, and for the
 *          variants without ET the factors are bit-identical to mla_getrf_la's;
 *          > 0 (default 4096): the factored columns are taken in super-blocks of `deep` columns, the rank-b updates
 *          stop at the super-block's last row and the rows below get ONE multiply of depth `deep` per super-block
 *          (34-35 TFLOP/s; same pivots, factors equal up to rounding). */
int mla_set_host_phases(mla_handle h, const int64_t* bounds, int count, int deep);

/* One update step of the multi-GPU driver as a single persistent launch: apply the broadcast panel P
 * (rows x w: unit-lower L11 on top of L21, leading dimension ldp) with its w panel-local pivots to the
 * column block T (rows x cols view starting at the panel's first row):
 *   T := interchanges(T);  T[0:w] := trilu(L11)^-1 T[0:w];  T[w:] -= L21 * T[0:w]
 * (laswp -> trsm_llu -> gemm_malleable of lu.py:251-253, 280-281, 289, 306-308).  Asynchronous. */
int mla_apply_panel(mla_handle h, const double* P, int64_t rows, int64_t w, int64_t ldp, double* T,
                    int64_t cols, int64_t ldt, const int32_t* ipiv, void* stream);

/* The two halves of mla_apply_panel.  prepare: interchange plan of the w pivots, inverses of the 128 x 128
 * diagonal blocks of the panel's unit-lower top block (the solves run in 128-row steps), empty work queue,
 * fresh step tag.  launch: `ctas` CTAs (0 = mla_set_update_sms / all) draining the prepared queue; a second
 * launch of the same step on another stream JOINS that queue (worker sharing across kernels: the SMs that
 * factored the next panel help with the update once the panel is done, pool.py:377-414).
 *   skip_cols: leading columns of T that already carry the interchanges and their U rows (leftover of an
 *              ET-cut panel, lu.py:247-255): they only take part in the rank-w update;
 *   L / left_cols / ldl: the owned columns LEFT of the panel (view starting at the panel's first row,
 *              nullable): they receive the interchanges only (lu.py:252, 329-332), as extra queue items.
 * The CTA that completes the step's last item publishes the step tag in the handle's step flag
 * (mla_step_flag) -- the ru_done of lu.py:309-310 for a panel kernel running beside the update. */
int mla_apply_panel_prepare(mla_handle h, const double* P, int64_t ldp, const int32_t* ipiv, int64_t w, int64_t rows,
                            void* stream);
int mla_apply_panel_launch(mla_handle h, const double* P, int64_t rows, int64_t w, int64_t ldp, double* T,
                           int64_t cols, int64_t ldt, int64_t skip_cols, double* L, int64_t left_cols, int64_t ldl,
                           int ctas, void* stream);

/* Device address of the handle's step flag and the tag of the step prepared last (mla_apply_panel_prepare):
 * *flag == tag  <=>  that step's queue has been drained.  Pass both to mla_panel_ll_async as the ET flag. */
int mla_step_flag(mla_handle h, uint32_t** flag_dev, uint32_t* tag);

/* Pack a factored panel for the broadcast of the multi-GPU driver: out receives
 *   [int32 x 4: factored width, singular flag, scheduled width w, rows][int32 x w panel-local pivots, padded
 *    to a multiple of 4][rows x w doubles, column-major, leading dimension rows]
 * = mla_packed_panel_doubles(rows, w) doubles.  use_panel_info != 0 takes the factored width and the
 * singular flag from the info record the last panel kernel of THIS handle left on the device (the chain
 * panel -> pack -> broadcast needs no host read-back); else they are w and 0.  Pivots travel as int32. */
int mla_pack_panel(mla_handle h, const double* P, int64_t rows, int64_t w, int64_t ld, const int32_t* ipiv,
                   int use_panel_info, double* out, void* stream);
int64_t mla_packed_panel_doubles(int64_t rows, int64_t w);

/* The device-side abort word of the handle (0 = no watchdog / protocol abort since the last launch that
 * reset it); the asynchronous entry points never read it back themselves.  Synchronises the device. */
int mla_abort_word(mla_handle h);

/* Number of SMs mla_apply_panel launches on (0 = all).  Lets a multi-GPU driver leave SMs to the
 * communication kernels or to the look-ahead panel (mla_panel_ll_async on another stream and another
 * handle) that runs beside the update. */
int mla_set_update_sms(mla_handle h, int ctas);

/* fill_random(a, seed) -- matrix.py:44-63: SplitMix64 stream, bit-identical to the reference;
 * value = scale*u + shift with u in (0,1) (scale=1, shift=0 reproduces fill_random; 2,-1 gives the
 * uniform[-1,1] configs).  col0/total_rows select a column block of a larger matrix (multi-GPU).
 * row_scale (device, nullable): value *= row_scale[i]. */
int mla_fill_random(mla_handle h, double* A, int64_t rows, int64_t cols, int64_t ld, uint64_t seed,
                    int64_t col0, int64_t total_rows, double scale, double shift,
                    const double* row_scale, void* stream);

/* Phase timers of the panel team (ns, accumulated by team rank 0): [0] trsm, [1] gemm/slab load,
 * [2] pivot steps, [3] write-back + swaps, [4] block barrier, [5] exchange share of [2].
 * Synchronises the device. */
int mla_panel_profile(mla_handle h, uint64_t* out16, int reset);

/* Device trace of the last mla_getrf_la call (the GPU analogue of the reference's Tracer,
 * trace.py:26-66): one row of 5 uint64 per outer iteration -- globaltimer ns of [0] iteration start,
 * [1] next panel's columns updated (panel may start), [2] panel end, [3] remainder update complete,
 * [4] scheduled width << 32 | factored width.  Returns the number of rows copied. Synchronises. */
int mla_getrf_trace(mla_handle h, uint64_t* out, int max_rows);

/* Per-CTA device trace -- the GPU form of the reference's Tracer (trace.py:26-66: one private event buffer
 * per worker, stamps from one clock).  After mla_set_trace(h, 1) every CTA of the persistent kernel appends
 * one record per phase it runs (thread 0, globaltimer stamps taken where the phase actually starts and ends):
 *   kind 1: drained the next panel's update queue (PF1/PF2 + RU helpers, lu.py:279-289)
 *   kind 2: factored the look-ahead panel as a member of the panel team (PF3, lu.py:291)
 *   kind 3: drained the remainder update queue as a member of the update team (RU1/RU2)
 *   kind 4: the same queue, entered by a panel-team CTA AFTER its panel ended (worker sharing, pool.py:377-414;
 *           the reference's MERGED team) -- stamped at the actual join
 *   kind 5: panel factored by the whole grid (prologue, and every panel of variant "lu")
 * mla_getrf_events copies max_per_cta records per CTA (unused records have kind 0) into out[cta][max_per_cta]
 * and returns the number of CTAs (0 when tracing is off).  Synchronises the device. */
typedef struct {
  uint64_t t_start, t_end;   /* globaltimer ns */
  int32_t iter;              /* outer iteration; 0 = prologue */
  int32_t kind;
  int32_t items;             /* queue items executed / panel columns factored */
  int32_t team;              /* CTAs in the panel team of that iteration */
} mla_trace_event;
int mla_set_trace(mla_handle h, int enable);
int mla_getrf_events(mla_handle h, mla_trace_event* out, int max_per_cta);

/* Time accounting of one update-team CTA during the last mla_getrf_la call (ns): [0] in GEMM tiles,
 * [1] tile count, [2] in PREP items, [3] PREP count, [4] in LEFT items, [5] iteration barriers +
 * bookkeeping, [6] whole kernel. */
int mla_getrf_debug(mla_handle h, uint64_t* out8);

/* residual_lu (matrix.py:116-131) has no entry point of its own: the Python layer composes it from
 * mla_laswp (P*A) and mla_gemm (blocked L*U), see paper_1611_06365_b200/matrix.py. */

#ifdef __cplusplus
}
#endif
#endif /* MLA_B200_H */
