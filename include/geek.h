/*
 * geek.h -- C ABI of libgeek.so, the B200 (sm_100a) kernels behind the GEEK
 * hot path: bucketize -> SILK seeding -> one-pass assignment.
 *
 * The reference (lshclust, pure Python + numpy) has no FFI; each entry point
 * below replaces the numpy inner loop cited beside it (paths relative to
 * /root/reference/pkg/src/lshclust).  The Python package
 * paper_2106_10515_b200 binds these with ctypes behind
 * the reference's own API names.
 *
 * Conventions
 *   - every pointer argument is a DEVICE pointer unless its name ends in
 *     `_host`; sizes are element counts; `stream` is a cudaStream_t (NULL =
 *     legacy default stream);
 *   - every function returns GEEK_OK (0) or a negative status and never
 *     throws; geek_last_error() describes the last failure of the calling
 *     host thread;
 *   - functions are stream-ordered and reentrant; a few (marked SYNC) read a
 *     data-dependent size back to the host and synchronise `stream`;
 *   - ids are uint32 (n < 2^32); MinHash values are uint32 (universe < 2^32).
 */
#ifndef GEEK_H
#define GEEK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GEEK_OK 0
#define GEEK_EINVAL -1 /* precondition violated (maps to InvalidInput) */
#define GEEK_ECUDA -2  /* CUDA runtime error (maps to EngineError)     */
#define GEEK_ENOMEM -3 /* device allocation failed                     */
#define GEEK_ERANGE -4 /* output capacity too small; size reported     */

#define GEEK_NONE 0xFFFFFFFFu /* "no value" for MinHash minima / codes */

/* One MinHash permutation pi over [0, u) (hashing.py:51-140).
 * u > 4096: cycle-walking w-bit mix, w = bitlen(u-1) <= 32, with
 *   mask, c1, c2, a1, s1, s2 exactly as hashing.py:97-113, and the inverse
 *   multipliers c1inv, c2inv (mod 2^w) for the inverse-rank scan.
 * u <= 4096: `table` is the offset of pi (u entries) inside the caller's
 *   table pool, `inv_table` the offset of pi^-1 (hashing.py:80-95);
 *   GEEK_NONE when mixing.                                                 */
typedef struct {
  uint64_t u;
  uint32_t mask, c1, c2, a1, s1, s2, c1inv, c2inv;
  uint32_t table, inv_table;
} geek_perm_t;

int geek_version(void);
const char* geek_last_error(void);
/* number of SMs of the current device, or a negative status */
int geek_device_sms(void);

/* ---- MinHash --------------------------------------------------------- */

/* out[p*count + i] = pi_p(x[i])   (MinHashFunction.permute, hashing.py:126-140) */
int geek_perm_forward(const geek_perm_t* perms_host, int nperm, const uint32_t* tables,
                      const uint32_t* x, uint64_t count, uint32_t* out, void* stream);

/* out[p*count + i] = pi_p^-1(r[i]), r[i] < universe (the bijection's inverse; the
 * inverse-rank scan's id lookup, hashing.py:97-140).  Used by the pipeline's
 * singleton-bucket bins: the object whose singleton bucket carries a signature. */
int geek_perm_inverse(const geek_perm_t* perms_host, int nperm, const uint32_t* tables,
                      const uint32_t* r, uint64_t count, uint32_t* out, void* stream);

/* sig[s*nperm + p] = min_{e in set s} pi_p(e); sets are CSR (flat, offsets[nsets+1]),
 * non-empty.  (SignatureScheme.signatures_for_sets, hashing.py:265-282)        */
int geek_set_minhash(const geek_perm_t* perms_host, int nperm, const uint32_t* tables,
                     const uint32_t* flat, const uint64_t* offsets, uint64_t nsets,
                     uint32_t* sig, void* stream);

/* Inverse-rank scan: for a family of m partitions of [0, n) given
 * id-major as codes[i*m + j] in [0, t), writes sig[p*(m*t) + j*t + s] =
 * min_{i : codes[i*m+j] == s} pi_p(i) for every non-empty bucket (GEEK_NONE
 * for empty ones).  `nonempty_host` (may be NULL: then every bucket is assumed
 * non-empty) gives the number of non-empty buckets the scan must cover.
 * Bit-identical to the member scan of engine.py:256-266.  SYNC.            */
int geek_silk_invscan(const uint32_t* codes, uint64_t n, int m, uint64_t t,
                      const geek_perm_t* perms_host, int nperm, const uint32_t* tables,
                      uint32_t* sig, const uint64_t* nonempty_host, uint64_t* draws_host,
                      void* stream);

/* ---- dense bucketize -------------------------------------------------- */

/* keys[j*n + i] = order-preserving uint64 image of the float64 projection
 * <x_i, A_j> (transform.py:125, engine.py:180); -0.0 folds onto +0.0 and NaN
 * onto the top key, matching np.lexsort.  dtype 0 = float32 X, 1 = float64.
 * `exprange` (device int[2], may be NULL; caller initialises {INT_MAX-ish,
 * INT_MIN-ish}) receives atomic min/max of the exact-sum exponent window of
 * X (as geek_exponent_range), fused into the same pass over X.  float32 rows
 * with d % 4 == 0, d <= 128 (and the digit tiles within SMEM: m <= 40 at
 * d = 128) run as exact integer-digit products on tcgen05 (kind::i8), keys
 * within the float64 order bound of the exact dot product; other shapes and
 * GEEK_TCPROJ=0 use float64 DMMA / FMA chains.                              */
int geek_project_keys(const void* X, int dtype, uint64_t n, int d, const double* A, int m,
                      uint64_t* keys, int* exprange, void* stream);

/* geek_project_keys for a shard of rows [row_lo, row_lo + n) of an ntot-row
 * job, with the bucket synchronisation fused in (engine.py:199-238): the key
 * of table j is stored straight into owner rank j % G's buffer,
 * dst_host[j % G][(j / G) * ntot + row_lo + i] -- device pointers that may be
 * peer (NVLink) mappings, e.g. a symmetric-memory buffer.  float32 X only,
 * d % 4 == 0, d <= 128, m <= 48, G <= 8.  The caller orders the ranks'
 * writes against the owners' reads (barrier before and after).             */
int geek_project_keys_routed(const void* X, int dtype, uint64_t n, int d, const double* A, int m,
                             uint64_t* const* dst_host, int G, uint64_t ntot, uint64_t row_lo, int* exprange,
                             const uint32_t* fine_cinfo, int cb, uint32_t* fine_cnt, void* stream);
/* ...and with fine_cnt != NULL it also performs the rank split's fine-bin
 * count of every key it writes: fine_cnt[f] += 1 for f = the key's fine bin
 * under fine_cinfo (uint2 [m][2^cb] from geek_fine_layout, global bins).    */

/* Precounted rank split (the fine histogram comes from the projection):
 *  geek_split_plan     coarse bits and sample stride of an n-key split;
 *  geek_coarse_hist    hist[j][cell] += sample keys [m][ns] (caller zeroes);
 *                      the sample is rows 0, stride, 2*stride, ... of the job;
 *  geek_fine_layout    fine bins of every cell from hist: cinfo (uint2
 *                      [m][2^cb] = {bins, first global bin}), toff[m+1] =
 *                      first global bin of each table, *nfb_host = total;
 *  geek_rank_split_counted  geek_rank_split of keys [m][n] given the tables'
 *                      hist rows [m][2^cb] and their fine counts concatenated
 *                      in table order.  SYNC.                               */
int geek_split_plan(uint64_t n, int* cb_out, uint64_t* stride_out);
int geek_coarse_hist(const uint64_t* keys, uint64_t ns, int m, int cb, uint32_t* hist, void* stream);
int geek_fine_layout(const uint32_t* hist, int m, uint64_t n, uint32_t* cinfo, uint32_t* toff, uint64_t* nfb_host,
                     void* stream);
int geek_rank_split_counted(const uint64_t* keys, uint64_t n, int m, uint64_t t, const uint32_t* hist,
                            const uint32_t* fcnt, uint32_t* codes, uint64_t* stats_host, void* stream);

/* Exact even rank split of every table (transform.py:95-109, engine.py:219-225):
 * codes[i*m + j] = slot of id i in table j, ties broken by id.  keys are
 * [m][n] as produced by geek_project_keys (or any order-preserving image).
 * stats_host[0..3] (may be NULL) = {fine bins, straddling ids, max straddle
 * bin, fallback sorts}.  SYNC.                                              */
int geek_rank_split(const uint64_t* keys, uint64_t n, int m, uint64_t t, uint32_t* codes,
                    uint64_t* stats_host, void* stream);

/* Rank-split boundary exceptions (north_star tie tolerance; transform.py:103-109
 * ranks OpenBLAS dgemv projections, engine.py:178-181).  For every table j and
 * bucket boundary s, midpoint = (max key of bucket s + min key of bucket s+1)/2;
 * counts[0] = ids whose key lies within tol_abs[j] (device double [m]) of a
 * neighbouring midpoint -- the only ids whose code may differ from the
 * reference's (a boundary whose two keys are equal is decided by id, so ids
 * holding exactly that key are not counted there); counts[1] / counts[2] = ids within rel_a / rel_b * |midpoint|;
 * counts[3] = entries offered to list.  list (device uint32 [cap][2]) receives
 * (table, id) of the tol_abs ids.  keys [m][n] as geek_project_keys writes
 * them, codes[i*code_stride + j] as geek_rank_split writes them.  Scratch:
 * workspace of geek_split_boundary_workspace(m, t) bytes.  Stream-ordered.  */
uint64_t geek_split_boundary_workspace(uint64_t m, uint64_t t);
int geek_split_boundary_stats(const uint64_t* keys, uint64_t n, int m, uint64_t t, const uint32_t* codes,
                              uint64_t code_stride, const double* tol_abs, double rel_a, double rel_b,
                              unsigned long long* counts, uint32_t* list, uint64_t cap, void* workspace,
                              uint64_t workspace_bytes, void* stream);

/* Same split for a single column of keys written with a row stride:
 * codes[i*stride + col] (used for numeric discretisation, transform.py:131-155). */
int geek_rank_split_strided(const uint64_t* keys, uint64_t n, uint64_t t, uint32_t* codes,
                            uint64_t stride, uint64_t col, void* stream);

/* order-preserving keys of a float64 / float32 column with a row stride */
int geek_column_keys(const void* values, int dtype, uint64_t n, uint64_t stride, uint64_t col,
                     uint64_t* keys, void* stream);

/* ---- sort / group-by primitives ---------------------------------------- */

/* Lexicographic stable sort of nrows rows of `width` uint32 columns
 * (row-major); perm[r] = original index of the r-th smallest row; gid[r] =
 * dense group index of that row (equal rows share it); *ngroups_host.
 * (np.unique(axis=0, return_inverse) + stable argsort: seeding.py:83-90,
 * transform.py:158-169).  `bits_host` (may be NULL) bounds each column. SYNC. */
int geek_group_rows(const uint32_t* rows, uint64_t nrows, int width, const int* bits_host,
                    uint32_t* perm, uint32_t* gid, uint64_t* ngroups_host, void* stream);

/* ---- SILK vote --------------------------------------------------------- */

/* Emit (bin, id) membership pairs for binned buckets of the id-major
 * partition `codes`: for each id i and table j with bucket b = j*t + code,
 * for each bin in bb_bins[bb_off[b] .. bb_off[b+1]) emit (bin, i).
 * *count_host returns the number written (capacity = cap).  SYNC.          */
int geek_emit_members_codes(const uint32_t* codes, uint64_t n, int m, uint64_t t,
                            const uint32_t* bb_off, const uint32_t* bb_bins,
                            uint32_t* out_bin, uint32_t* out_id, uint64_t cap,
                            uint64_t* count_host, void* stream);

/* Fused emission + strict-majority vote over an id-major partition: an id's
 * multiplicity in a bin is read off its own code row, so only winning (bin,
 * id) pairs are written (unique, unordered).  GEEK_ERANGE when an id reaches
 * more than 64 bins (callers fall back to the pair path).  SYNC.           */
int geek_emit_winners_codes(const uint32_t* codes, uint64_t n, int m, uint64_t t,
                            const uint32_t* bb_off, const uint32_t* bb_bins, const uint32_t* bin_size,
                            uint32_t* out_bin, uint32_t* out_id, uint64_t cap,
                            uint64_t* count_host, void* stream);

/* Winners grouped by bin, ids ascending, bins with < delta winners dropped
 * (seeding.py:160, engine.py:281).  id_bound bounds the ids.  SYNC.        */
int geek_group_winners(const uint32_t* win_bin, const uint32_t* win_id, uint64_t nwin, uint64_t nbins,
                       uint64_t id_bound, uint64_t delta, uint32_t* out_bin, uint32_t* out_id,
                       uint64_t* nout_host, void* stream);

/* Strict-majority vote (seeding.py:107-114, engine.py:278-282): given (bin,
 * id) pairs (any order; a bucket listed once per bin) and bin sizes in
 * buckets, writes the winners grouped by bin with ids ascending
 * (win_bin/win_id, *nwin_host) after dropping bins with < delta winners.
 * SYNC.                                                                    */
int geek_majority_vote(const uint32_t* pair_bin, const uint32_t* pair_id, uint64_t npairs,
                       const uint32_t* bin_size, uint64_t nbins, uint64_t delta,
                       uint32_t* win_bin, uint32_t* win_id, uint64_t* nwin_host,
                       void* stream);

/* ---- dedup helpers ----------------------------------------------------- */

/* Given groups (CSR flat/offsets) and a grouping of them into bins (perm/gid
 * from geek_group_rows over their signatures), keep[g] = 1 for the one
 * representative per bin: largest, ties to the lexicographically smallest
 * member sequence (seeding.py:117-134).                                    */
int geek_pick_representatives(const uint32_t* flat, const uint64_t* offsets, const uint32_t* perm,
                              const uint32_t* gid, uint64_t ngroups, uint8_t* keep, void* stream);

/* Canonical order of groups by member tuple (SeedGroup.key, data.py:200-202;
 * a proper prefix sorts first): order[r] = index of the r-th group.  SYNC. */
int geek_sort_groups(const uint32_t* flat, const uint64_t* offsets, uint64_t ngroups,
                     uint32_t* order, void* stream);

/* ---- exact centers ----------------------------------------------------- */

/* min / max binary exponent over the non-zero entries of X (frexp sense);
 * out_host = {emin, emax} (emin > emax when X is all zero).  SYNC.          */
int geek_exponent_range(const void* X, int dtype, uint64_t n, int d, int* out_host, void* stream);

/* Exact per-group column sums in base-2^32 digits relative to 2^emin
 * (numeric.py:19-40): digits[(g*d + c)*nd + k] (int64, ADDED to).  Members
 * are global ids; rows outside [row_lo, row_lo + nrows) are skipped (a shard
 * contributes only its own rows; engine.py:299-311).  *nonfinite (device,
 * may be NULL) is OR-ed with 1 when a member coordinate is NaN / inf -- the
 * reference raises ValueError("non-finite value in exact sum") there
 * (numeric.py:24-25).  Stream-ordered (chunk table built on the device).    */
int geek_exact_sums(const void* X, int dtype, uint64_t nrows, int d, uint64_t row_lo,
                    const uint32_t* flat, const uint64_t* offsets, uint64_t ngroups,
                    int emin, int nd, int64_t* digits, unsigned* nonfinite, void* stream);

/* Transport accounting of the reference's LocalCenters message
 * (serialize.py pack_center_stats -> numeric.py pack_bigints): *out (device)
 * += sum over (group, column) of 8 + (bitlen|T| + 8) / 8 + 1 bytes, where
 * T = S * 2^(emin + 1074) is the reference's scaled-integer sum of the digit
 * sums S.  Stream-ordered.                                                  */
int geek_sum_pack_bytes(const int64_t* digits, uint64_t ngroups, int d, int nd, int emin,
                        unsigned long long* out, void* stream);

/* Correctly rounded means from the digit sums (numeric.py:43-46).           */
int geek_round_means(const int64_t* digits, const uint64_t* counts, uint64_t ngroups, int d,
                     int emin, int nd, double* out, void* stream);

/* ---- assignment -------------------------------------------------------- */

/* Statistics of one geek_assign_l2 call, written on the device (stream-ordered;
 * replaces round 1's process-global geek_assign_last_* counters).           */
typedef struct {
  unsigned long long rechecked;   /* points re-evaluated exactly (screen candidates + full scans) */
  unsigned long long full_scans;  /* of those, points whose candidate window overflowed: all centers */
  unsigned long long screen_mode; /* 16 FP16x3, 3 TF32x3 (also after an f16 overflow), 17 tile-local
                                     FP16, 1 TF32, 0 no tensor-core screen */
  unsigned long long screen_tiles; /* FP16x3 screen: (point tile, center tile) pairs multiplied --
                                     the rest were skipped as out of reach (0 for other screens) */
} geek_assign_stats_t;

/* Nearest center by float64 direct-difference distance with numpy's pairwise
 * summation order and first-index ties (assignment.py:54-62, :95-99):
 * labels[i], best[i] = distance.  C is [k][d] float64.  float32 X with
 * d <= 128 and k >= 4 goes through the tcgen05 screen (FP16x3; env
 * GEEK_SCREEN=17 / 3 / 1 selects tile-local FP16 / TF32x3 / TF32) and an
 * exact float64 recheck.  Fully stream-ordered (no host synchronisation):
 *   stats (device, may be NULL)       receives geek_assign_stats_t;
 *   ev_screen_begin / ev_screen_end   (cudaEvent_t, may be NULL) are recorded
 *                                     around the screen launches, so the
 *                                     caller can time the dominant kernel;
 *   workspace / workspace_bytes       caller scratch of at least
 *                                     geek_assign_l2_workspace_size(n, d, k)
 *                                     bytes; NULL = the stream-ordered pool;
 *                                     too small -> GEEK_ERANGE.            */
uint64_t geek_assign_l2_workspace_size(uint64_t n, int d, uint64_t k);
int geek_assign_l2(const void* X, int dtype, uint64_t n, int d, const double* C, uint64_t k,
                   int64_t* labels, double* best, geek_assign_stats_t* stats, void* ev_screen_begin,
                   void* ev_screen_end, void* workspace, uint64_t workspace_bytes, void* stream);

/* Self-test of the tcgen05 screen on a synthetic problem (1000 x 128
 * points, 300 centers): out_host[0] = max |s_tc - S_f64| / (|x'||c'|max)
 * over every kept entry, out_host[1] = points whose screened top-1 is not
 * the f64 argmin.  lbo/sbo are the canonical-layout core-matrix strides in
 * bytes; nprod = 1 (TF32), 3 (TF32x3), 16 (FP16x3 over power-of-two
 * scaled operands, the default screen of geek_assign_l2) or 17 (tile-local
 * FP16).  SYNC (test entry point).                                          */
int geek_tc_selftest(uint32_t lbo, uint32_t sbo, int nprod, double* out_host);

/* radii[c] = max best over members (0 if none), sizes[c] = member count
 * (assignment.py:100-101, data.py:243-245).  Accumulates (call on zeroed
 * outputs, or on partial results to merge).                                 */
int geek_radii_sizes(const int64_t* labels, const double* best, uint64_t n, uint64_t k,
                     double* radii, int64_t* sizes, void* stream);

/* numpy pairwise sum (float64 add.reduce) of v[0..n): *out (device).        */
int geek_pairwise_sum(const double* v, uint64_t n, double* out, void* stream);

/* Jaccard assignment, categorical records (assignment.py:63-67):
 * dist = 1 - m/(2d - m), m = #equal attributes; codes [n][d], modes [k][d]. */
int geek_assign_categorical(const int32_t* codes, uint64_t n, int d, const int32_t* modes,
                            uint64_t k, int64_t* labels, double* best, void* stream);

/* Jaccard assignment, sparse sets vs binary modes (assignment.py:68-78);
 * sets are CSR over [0, universe); modes are [k][universe] int32 0/1.       */
int geek_assign_sparse(const uint32_t* flat, const uint64_t* offsets, uint64_t n,
                       uint64_t universe, const int32_t* modes, uint64_t k, int64_t* labels,
                       double* best, void* stream);

/* ---- sparse / categorical helpers --------------------------------------- */

/* DOPH reduction (hashing.py:312-329): per set, tokens (bin + (min rel mod
 * 2^61-1)) mod r, sorted unique, written to out_flat at offsets
 * out_off[s]..; out_off must be sized by geek_doph_reduce's first call
 * (out_flat NULL => only counts[s] are written).                            */
int geek_doph_reduce(const geek_perm_t* perm_host, const uint32_t* tables, const uint32_t* flat,
                     const uint64_t* offsets, uint64_t nsets, uint64_t D, uint64_t r,
                     uint32_t* counts, const uint64_t* out_off, uint32_t* out_flat, void* stream);

/* Mode statistics: counts[(g*d + c)*cs + v] += #members of group g whose
 * column c equals v (seeding.py:180-185, engine.py:312-317).                */
int geek_mode_counts(const int32_t* codes, uint64_t nrows, int d, uint64_t row_lo, uint64_t cs,
                     const uint32_t* flat, const uint64_t* offsets, uint64_t ngroups,
                     int64_t* counts, void* stream);

/* Sparse membership counts: counts[g*universe + e] += #members containing e. */
int geek_sparse_counts(const uint32_t* set_flat, const uint64_t* set_off, uint64_t nrows,
                       uint64_t row_lo, uint64_t universe, const uint32_t* flat,
                       const uint64_t* offsets, uint64_t ngroups, int64_t* counts, void* stream);

/* ---- refinement passes (assignment.py:110-170, engine.py:519-537) ------ */

/* Exact digit column sums keyed by label: digits[(labels[i]*d + c)*nd + q]
 * += row i's column c in base-2^32 digits relative to 2^emin (the
 * geek_exact_sums representation; ADDED to, so shards reduce by addition).
 * Rows stream once in storage order (order NULL) or in the order of the row
 * permutation `order` (e.g. sorted by label, so equal labels form register
 * runs); labels outside [0, k) are skipped.  ASYNC.                         */
int geek_label_sums(const void* X, int dtype, uint64_t nrows, int d, const int64_t* labels,
                    const int64_t* order, uint64_t k, int emin, int nd, int64_t* digits, void* stream);

/* counts[(labels[i]*d + c)*cs + codes[i*d + c]] += 1 (categorical modes of
 * the current clusters, assignment.py:122-126).  ASYNC.                      */
int geek_label_mode_counts(const int32_t* codes, uint64_t nrows, int d, const int64_t* labels, uint64_t k,
                           uint64_t cs, int64_t* counts, void* stream);

/* counts[labels[i]*universe + e] += 1 for every e in set i (sparse modes of
 * the current clusters, assignment.py:127-131).  ASYNC.                      */
int geek_label_sparse_counts(const uint32_t* set_flat, const uint64_t* set_off, uint64_t nrows,
                             const int64_t* labels, uint64_t k, uint64_t universe, int64_t* counts,
                             void* stream);

/* ---- ingestion (io.py:21-48) -------------------------------------------- */

/* Strip nrec .fvecs (elem_bytes 4) / .bvecs (elem_bytes 1) records of
 * dimension d from device memory `raw` into float32 out[nrec][d];
 * *bad_rec (device, caller-initialised to UINT64_MAX) is lowered to the
 * first record whose 4-byte prefix is not d.  ASYNC.                       */
int geek_unpack_vecs(const void* raw, uint64_t nrec, int d, int elem_bytes, float* out, uint64_t* bad_rec,
                     void* stream);

/* ---- artifacts (serialize.py:129-162) ------------------------------------ */

/* Byte image of lshclust.serialize.dump_buckets' bucket records at out + base:
 * bucket b (table t with table_off[t] <= b < table_off[t+1], slot b -
 * table_off[t]) takes 34 + 8*size bytes starting at base + 34*b + 8*offsets[b]
 * (<q table><q slot><q length><B 1><B 1><q size> + int64 ids, little-endian).
 * table_off is a device array of ntables+1 entries.  ASYNC.                  */
int geek_pack_buckets(const uint32_t* flat, const uint64_t* offsets, const uint64_t* table_off, int ntables,
                      uint64_t nbuckets, uint64_t base, uint8_t* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GEEK_H */
