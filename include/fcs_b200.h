/*
 * fcs_b200.h — C-ABI of the B200-native fast count sketch (FCS) library.
 *
 * This is the drop-in boundary for the FCS hot path of the reference
 * (`/root/reference/proj`, namespace `sketchtensor`). Every entry point takes
 * plain pointers and sizes (no torch, Eigen or C++ types) and names the
 * reference interface it replaces as file:line. Unless marked HOST, tensor /
 * table / output pointers are DEVICE pointers on the current CUDA device and
 * work is stream-ordered on `stream` (a cudaStream_t, NULL = legacy default).
 *
 * Errors: every int-returning call returns one of the ST_* codes below.
 * ST_EINVAL mirrors the reference's std::invalid_argument (validation is on
 * the host, before any launch); ST_ENUMERIC mirrors std::runtime_error
 * (idft_real's imaginary-residue check, fft.cpp:69-71). st_last_error()
 * returns the thread's last message (same text as the reference where one
 * exists). There is no CPU fallback: with no usable GPU every compute entry
 * fails with ST_ECUDA.
 *
 * Table layout ("packed family tables"): for D families over N modes with
 * dims I_0..I_{N-1}, entry (d, n, i) lives at
 *     packed[d * sum(I) + (I_0 + ... + I_{n-1}) + i]
 * as  bucket | (sign < 0 ? 1u << 31 : 0)   (bucket < 2^31).
 * Dense tensors are column-major, first index fastest (tensor.hpp:10-13).
 * Sketch outputs are fp64, D rows of J~ = sum(J_n) - N + 1, row-major.
 */
#ifndef FCS_B200_H
#define FCS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ST_OK = 0,
  ST_EINVAL = 1,   /* std::invalid_argument in the reference */
  ST_ENUMERIC = 2, /* std::runtime_error (idft_real residue) */
  ST_ECUDA = 3,
  ST_ENCCL = 4,
  ST_ENOMEM = 5
};

enum { ST_F32 = 0, ST_F64 = 1 };

/* SketchKind (sketch.hpp:10), same order. */
enum { ST_SKETCH_CS = 0, ST_SKETCH_TS = 1, ST_SKETCH_FCS = 2 };

/* SketchBackend (cpd.hpp:13), same order. */
enum {
  ST_BACKEND_PLAIN = 0,
  ST_BACKEND_CS = 1,
  ST_BACKEND_TS = 2,
  ST_BACKEND_HCS = 3,
  ST_BACKEND_FCS = 4
};

#define ST_MAX_ORDER 8

/* Thread-local text of the last failure. */
const char* st_last_error(void);
/* ABI version of this header (bumped on any signature change). */
int st_abi_version(void);
/* Device facts used for grid sizing: SM count, opt-in smem per block, L2. */
int st_device_query(int* sm_count, size_t* smem_optin, size_t* l2_bytes);

/* ------------------------------------------------------------------ hashing */

/* HOST. family_seed(base, d) = SplitMix64::mix(base + d).
 * Replaces sketchtensor::family_seed, hashing.cpp:123-125. */
uint64_t st_family_seed(uint64_t base_seed, size_t d);

/* K0. Tabulates HashPair(input_dim, hash_len, seed) on the device: bucket[i]
 * from draw 2i+1 (Lemire mulhi), sign[i] from the top bit of draw 2i+2,
 * bit-exact with the serial host stream.
 * Replaces HashPair::HashPair(size_t, size_t, uint64_t), hashing.cpp:10-22. */
int st_hash_tabulate(uint64_t seed, size_t input_dim, size_t hash_len, uint32_t* bucket,
                     int8_t* sign, void* stream);

/* K0 over a whole estimator configuration: D families (master seed
 * master_seeds[d], pair n seeded master ^ n), written as packed tables.
 * Replaces HashFamily(dims, hash_lens, master), hashing.cpp:42-54, and
 * families_for, estimators.cpp:104-115 (callers pass family_seed(seed, d)). */
int st_family_tables(size_t order, const size_t* dims, const size_t* hash_lens,
                     size_t sketch_count, const uint64_t* master_seeds /* HOST */,
                     uint32_t* packed, void* stream);

/* Packs explicit (hand-built) device tables bucket[total], sign[total] into
 * packed form; validates bucket < hash_len per mode on the host side caller.
 * Serves HashPair(bucket_map, sign_map, hash_len), hashing.cpp:24-40. */
int st_pack_tables(size_t total, const uint32_t* bucket, const int8_t* sign, uint32_t* packed,
                   void* stream);

/* ------------------------------------------------------------- dense FCS */

/* Workspace bytes st_fcs_dense needs for this problem (0 if none). */
size_t st_fcs_dense_workspace(int dtype, size_t order, const size_t* dims, size_t last_count,
                              size_t sketch_count, const size_t* hash_lens);

/* K1. Dense FCS of a column-major order-N tensor for D families at once:
 *   out[d][sum_n h_{d,n}(i_n)] (+)= prod_n s_{d,n}(i_n) * T[i]
 * over every element; exact zeros contribute nothing (sketch.cpp:48-61).
 * `tensor` holds the slab i_{N-1} in [last_begin, last_begin + last_count)
 * of the full tensor `dims` (contiguous because the last mode is slowest) —
 * the shard a rank owns under element sharding; pass 0 / dims[N-1] for the
 * whole tensor. Numerics: dtype ST_F32 with I_0 % 4 == 0, I_0 <= 1024 and a
 * 16-byte aligned tensor accumulates each CTA's partial sketch in int32 fixed
 * point, value * 2^S rounded to nearest, with S chosen per call from a
 * sampled bound on the partials (error <= 2^-(S+1) per element; the same S
 * and result on every run). A CTA that meets an element out of range or
 * non-finite redoes its chunk in fixed point with those elements diverted to
 * an exact fp64 reduction; a partial reaching 2^30, or partials that all stay
 * below 2^16, make it redo the chunk with fp32 shared-memory atomics
 * (order-dependent rounding). Other fp32 shapes with I_0 <= 16384 and >= 8M
 * element-updates take the same int32 fixed point with scalar loads (fibers
 * longer than 1024 split into warp segments, sketches wider than shared
 * memory into bucket ranges; a flagged CTA redoes its chunk or range with
 * fp32 atomics); the rest accumulate in atomics.
 * ST_F64 with I_0 <= 16384 and >= 8M element-updates accumulates in 64-bit
 * fixed point (two int32 atomics per element, exact carries; partials summed
 * exactly in 128-bit integers; deterministic; a sketch wider than shared
 * memory is split into bucket ranges, one CTA each; a CTA that meets an
 * element out of range redoes its chunk with fp64 atomics), smaller calls in
 * fp64 atomics.
 * Partials are reduced in a fixed order. accumulate != 0 adds to out instead
 * of overwriting it.
 * Replaces fcs_sketch(const DenseTensor&, const HashFamily&), sketch.cpp:187-201
 * (D calls, one per family). */
int st_fcs_dense(int dtype, const void* tensor, size_t order, const size_t* dims,
                 size_t last_begin, size_t last_count, size_t sketch_count,
                 const uint32_t* packed, const size_t* hash_lens, double* out, int accumulate,
                 void* workspace, size_t workspace_bytes, void* stream);

/* HOST, synchronous diagnostics of the last st_fcs_dense call of this dtype
 * and shape that used `workspace`: the fixed-point exponent S (INT_MIN when
 * that call did not take a fixed-point kernel), the number of (chunk,
 * family) CTAs that fell back to float atomics, and the number of CTAs. */
int st_fcs_dense_report(int dtype, size_t order, const size_t* dims, size_t last_count,
                        size_t sketch_count, const size_t* hash_lens, const void* workspace,
                        size_t workspace_bytes, int* fx_exponent, size_t* fallback_ctas,
                        size_t* ctas);

/* HOST-buffer convenience: K0 on the device from the seeds, then the host
 * tensor (the slab [last_begin, last_begin + last_count) of the last mode of
 * `dims`; pass 0 / dims[N-1] for the whole tensor) is copied H2D in chunks on
 * one stream while K1 sketches the previous chunk on another, then the
 * D x J~ result is copied D2H; synchronised. Device buffers are cached per
 * device between calls. With pinned host memory the copies run at full link
 * speed. The end-to-end call a reference caller makes.
 * Replaces D x fcs_sketch(DenseTensor(dims, data), HashFamily(dims, J, seeds[d])). */
int st_fcs_dense_host(int dtype, const void* host_tensor, size_t order, const size_t* dims,
                      size_t last_begin, size_t last_count, size_t sketch_count,
                      const uint64_t* master_seeds, const size_t* hash_lens, double* host_out);

/* st_fcs_dense_host with explicit HOST packed tables (D families in the
 * packed layout above, e.g. hand-built pairs, hashing.cpp:24-40) instead of
 * master seeds. Replaces D x fcs_sketch(DenseTensor(dims, data), family_d). */
int st_fcs_dense_host_tables(int dtype, const void* host_tensor, size_t order,
                             const size_t* dims, size_t last_begin, size_t last_count,
                             size_t sketch_count, const uint32_t* host_packed,
                             const size_t* hash_lens, double* host_out);

/* Sparse-input FCS (north_star (1), O(nnz)): nnz nonzeros of
 * an order-N tensor of shape dims as COO — values[k] (ST_F32 / ST_F64) at
 * coords[k * order + n] (uint32, device) — for D families at once, out
 * (+)= D x J~ fp64 (device). Equal to fcs_sketch(DenseTensor) of the
 * densified tensor (sketch.cpp:187-201; duplicate coordinates add up, zeros
 * are skipped like for_each_nonzero, sketch.cpp:48-61). Coordinates out of
 * range are skipped and counted into *invalid (device, may be NULL): the
 * caller raises compose's "compose: index out of range" (hashing.cpp:90-92).
 * fp64 global reductions: run-to-run differences at the last bit. */
int st_fcs_coo(int dtype, const void* values, const uint32_t* coords, size_t nnz, size_t order,
               const size_t* dims, size_t sketch_count, const uint32_t* packed,
               const size_t* hash_lens, double* out, int accumulate,
               unsigned long long* invalid, void* stream);

/* Count sketch of R columns (cs_sketch_columns, sketch.cpp:118-133; R = 1 is
 * cs_sketch, sketch.cpp:105-116): u is I x R column-major (device), table is
 * one packed pair, out is hash_len x R column-major fp64 (overwritten). */
int st_cs_columns(const double* u, size_t input_dim, size_t cols, const uint32_t* packed_pair,
                  size_t hash_len, double* out, void* stream);

/* Read-out through one packed pair: out[l] = s(l) * src[h(l)], l < count
 * (device). Serves the free-mode readout sign_f(i) z[bucket_f(i)] of the
 * estimators (estimators.cpp:84-88,262-266) and the long-pair sketch's
 * virtual tensor s(l) sk[h(l)] (estimators.cpp:290-350). */
int st_cs_expand(const double* src, size_t src_len, const uint32_t* packed_pair, size_t count,
                 double* out, void* stream);

/* --------------------------------------------------------------- CP-form FCS */

/* Workspace bytes for st_fcs_cp. */
size_t st_fcs_cp_workspace(size_t order, const size_t* dims, size_t rank, size_t sketch_count,
                           const size_t* hash_lens);

/* K2-K5. FCS of a CP tensor sum_r w_r u_r^(1) o ... o u_r^(N) for D families:
 * per (d, r) the mode sketches CS_n(U^(n)[:, r]) are transformed, multiplied
 * pointwise, weighted and summed over r in the frequency domain, then one
 * inverse transform per d gives the length-J~ linear convolution. Only ranks
 * [r_begin, r_begin + r_count) are included (rank sharding); zero weights
 * are skipped like the reference. factors[n] is a device I_n x R column-major
 * fp64 matrix; weights is a device R-vector. accumulate != 0 adds into out.
 * Replaces fcs_sketch(const CpTensor&, const HashFamily&), sketch.cpp:203-207
 * (convolved_cp_sketch :65-86, fft_convolve fft.cpp:75-84). */
int st_fcs_cp(const double* weights, size_t rank, size_t order, const size_t* dims,
              const double* const* factors /* HOST array of device ptrs */, size_t r_begin,
              size_t r_count, size_t sketch_count, const uint32_t* packed,
              const size_t* hash_lens, double* out, int accumulate, void* workspace,
              size_t workspace_bytes, void* stream);

/* Linear convolution of two batched real sequences (D rows each):
 * out[d] = a[d] (*) b[d], length la + lb - 1. Serves the Kronecker path
 * (FCS(A (x) B) = FCS(A) (*) FCS(B)) and fft_convolve with
 * two inputs, fft.cpp:75-84. */
int st_convolve_pairs(const double* a, size_t la, const double* b, size_t lb, size_t batch,
                      double* out, void* stream);

/* ---------------------------------------------- exact-length transforms */

/* Forward DFT of a real device vector x (len entries) zero-padded or
 * truncated to EXACTLY n points: out (device, 2n doubles, interleaved
 * re/im) = sum_j x_j exp(-2 pi i jk / n), unnormalised. Bluestein chirp-z over
 * the library's shared-memory / two-level FFTs at a smooth length >= 2n - 1.
 * n = 0 -> ST_EINVAL "dft: zero length".
 * Replaces dft(std::span<const double>, size_t), fft.cpp:42-51. */
int st_dft(const double* x, size_t len, size_t n, double* out, void* stream);

/* Inverse of an n-bin device spectrum (2n doubles): out (device, n) = Re of
 * (1/n) sum_k X_k exp(+2 pi i jk / n). check != 0 makes the call synchronous
 * and returns ST_ENUMERIC "idft_real: inverse transform is not real" when
 * ||Im|| > 1e-9 ||Re|| + 1e-12, like the reference.
 * Replaces idft_real(const std::vector<std::complex<double>>&), fft.cpp:53-73. */
int st_idft_real(const double* spectrum, size_t n, double* out, int check, void* stream);

/* F^-1(F(x_1, n) ... F(x_k, n)) at exactly n points (circular convolution;
 * linear when n >= sum(len) - k + 1). inputs: HOST array of k device
 * pointers; lens: HOST; out: device n. Synchronous (residue check).
 * Replaces fft_convolve, fft.cpp:75-84. */
int st_fft_convolve(const double* const* inputs, const size_t* lens, size_t k, size_t n,
                    double* out, void* stream);

/* Cross-correlation vector z (device, n) of one precomputed FCS: the exact
 * n-point spectrum (device, 2n doubles, as st_dft returns for the sketch),
 * the count sketches of a (la entries) and b (lb) under the two contracted
 * modes' packed pairs (device, ja / jb buckets):
 *   z = idft_real(S conj(F cs_a) conj(F cs_b)). Synchronous (residue check).
 * Replaces precompute_z(const PrecomputedFcs&, a, b, free_mode),
 * estimators.cpp:151-167 (the caller picks the pairs by free_mode). */
int st_precompute_z(const double* spectrum, size_t n, const double* a, size_t la,
                    const uint32_t* pair_a, size_t ja, const double* b, size_t lb,
                    const uint32_t* pair_b, size_t jb, double* z, void* stream);

/* Kronecker-product compression (BASELINE config 5): for D 4-mode families
 * (pairs p0..p3 over dims ra, ca, rb, cb) returns FCS of the outer-product
 * tensor A o B = conv(FCS_{p0,p1}(vec A), FCS_{p2,p3}(vec B)), D x J~.
 * Composition of fcs_sketch(tensor_from_matrix(.)) (sketch.cpp:187-201,
 * tensor.cpp:272-276) and fft_convolve (fft.cpp:75-84). */
int st_fcs_kron(const double* a, size_t ra, size_t ca, const double* b, size_t rb, size_t cb,
                size_t sketch_count, const uint32_t* packed, const size_t* hash_lens,
                double* out, void* stream);

/* ------------------------------------------------------ TS and HCS sketches */

/* Tensor sketch of a dense tensor: bucket (sum_n h_n) mod J, all J_n equal
 * (else ST_EINVAL "ts_sketch: all hash lengths must be equal"); out is D x J.
 * Computed as the J-periodic fold of the dense FCS.
 * Replaces ts_sketch(const DenseTensor&, const HashFamily&), sketch.cpp:135-149. */
size_t st_ts_dense_workspace(int dtype, size_t order, const size_t* dims, size_t last_count,
                             size_t sketch_count, const size_t* hash_lens);
int st_ts_dense(int dtype, const void* tensor, size_t order, const size_t* dims, size_t last_begin,
                size_t last_count, size_t sketch_count, const uint32_t* packed,
                const size_t* hash_lens, double* out, int accumulate, void* workspace,
                size_t workspace_bytes, void* stream);

/* Tensor sketch of a CP tensor: circular convolution at length J of the
 * factor count sketches (= fold of the CP-form FCS); out is D x J.
 * Replaces ts_sketch(const CpTensor&, const HashFamily&), sketch.cpp:151-155. */
size_t st_ts_cp_workspace(size_t order, const size_t* dims, size_t rank, size_t sketch_count,
                          const size_t* hash_lens);
int st_ts_cp(const double* weights, size_t rank, size_t order, const size_t* dims,
             const double* const* factors /* HOST array of device ptrs */, size_t r_begin,
             size_t r_count, size_t sketch_count, const uint32_t* packed,
             const size_t* hash_lens, double* out, int accumulate, void* workspace,
             size_t workspace_bytes, void* stream);

/* Higher-order count sketch of a dense tensor into a J_0 x ... x J_{N-1}
 * column-major tensor per family (D x prod J_n doubles, prod J_n < 2^31).
 * Replaces hcs_sketch(const DenseTensor&, const HashFamily&), sketch.cpp:157-173. */
size_t st_hcs_dense_workspace(int dtype, size_t order, const size_t* dims, size_t last_count,
                              size_t sketch_count, const size_t* hash_lens);
int st_hcs_dense(int dtype, const void* tensor, size_t order, const size_t* dims,
                 size_t last_begin, size_t last_count, size_t sketch_count, const uint32_t* packed,
                 const size_t* hash_lens, double* out, int accumulate, void* workspace,
                 size_t workspace_bytes, void* stream);

/* Higher-order count sketch of a CP tensor: sum_r w_r CS_0(u_r) o ... o CS_{N-1}(u_r)
 * (zero weights skipped), D x prod J_n.
 * Replaces hcs_sketch(const CpTensor&, const HashFamily&), sketch.cpp:175-185. */
size_t st_hcs_cp_workspace(size_t order, const size_t* dims, size_t rank, size_t sketch_count,
                           const size_t* hash_lens);
int st_hcs_cp(const double* weights, size_t rank, size_t order, const size_t* dims,
              const double* const* factors /* HOST array of device ptrs */, size_t sketch_count,
              const uint32_t* packed, const size_t* hash_lens, double* out, int accumulate,
              void* workspace, size_t workspace_bytes, void* stream);

/* --------------------------------------------- sketched contraction engine */

typedef struct st_engine st_engine;

/* Builds D FCS sketches of an order-3 device tensor and caches their
 * spectra on the device (FcsEngine ctor, cpd.cpp:63-67 -> families_for +
 * precompute_fcs, estimators.cpp:104-115,140-149). The tensor is consumed
 * once and not retained. */
int st_engine_create(st_engine** engine, int dtype, const void* tensor, const size_t* dims,
                     size_t hash_len, size_t sketch_count, uint64_t seed, void* stream);
/* make_contraction_engine(t, backend, cfg) (cpd.cpp:220-232), every backend:
 * ST_BACKEND_FCS (FcsEngine, cpd.cpp:61-94), ST_BACKEND_TS (TsEngine,
 * cpd.cpp:96-126: D tensor sketches of length J, estimates by circular
 * correlation at length J, estimators.cpp:209-233), ST_BACKEND_PLAIN
 * (PlainEngine, cpd.cpp:36-59: exact contractions of a device copy of the
 * tensor; D is 1, no median), ST_BACKEND_HCS (HcsEngine, cpd.cpp:128-158:
 * D J x J x J sketches) and ST_BACKEND_CS (CsEngine, cpd.cpp:160-197: D
 * long-pair count sketches of vec(T)). st_engine_create == ST_BACKEND_FCS. */
int st_engine_create_backend(st_engine** engine, int backend, int dtype, const void* tensor,
                             const size_t* dims, size_t hash_len, size_t sketch_count,
                             uint64_t seed, void* stream);
/* An engine over GIVEN sketches instead of a tensor: D device rows of
 * composed length 3J - 2 (ST_BACKEND_FCS: the sketches of PrecomputedFcs,
 * estimators.cpp:140-145) or J (ST_BACKEND_TS: PrecomputedTs), the D
 * families' device packed tables over dims (all hash lengths J). Serves
 * estimate_uvw / estimate_iuv(std::span<const PrecomputedFcs / Ts>, ...),
 * estimators.cpp:169-191,219-233, for callers that hold sketches. */
int st_engine_from_sketches(st_engine** engine, int backend, const double* sketches,
                            size_t sketch_count, const size_t* dims, size_t hash_len,
                            const uint32_t* packed, void* stream);
int st_engine_destroy(st_engine* engine);
int st_engine_backend(const st_engine* engine);
/* Sketch length (J~ FCS, J TS and CS, J^3 HCS; 0 Plain) and the current
 * D x length sketch values (device out; ST_EINVAL for Plain). */
size_t st_engine_composed_len(const st_engine* engine);
int st_engine_sketches(st_engine* engine, double* out, void* stream);

/* Batched T(I, a, b) with the identity at free_mode: for each of `batch`
 * vector pairs (rows of a: batch x I_c1, rows of b: batch x I_c2, device
 * fp64) the median over D of s_f(i) * z_d[h_f(i)], z_d = IFFT(S_d conj(F cs_a)
 * conj(F cs_b)); out is batch x I_free. median != 0 applies median_reduce;
 * median == 0 writes all D estimates (batch x D x I_free) instead.
 * Replaces ContractionEngine::iuv / FcsEngine::iuv, cpd.cpp:74-77 ->
 * estimate_iuv, estimators.cpp:180-186 (iuv_spectral :66-90, median :125-138). */
int st_engine_iuv(st_engine* engine, size_t batch, const double* a, const double* b,
                  size_t free_mode, double* out, int median, void* stream);

/* Batched T(u, v, w): out[k] = median over D of (1/n) sum Re(S conj(G)).
 * Replaces FcsEngine::uvw, cpd.cpp:69-72 -> estimate_uvw, estimators.cpp:169-174
 * (uvw_spectral :48-64, spectral_dot :38-45). */
int st_engine_uvw(st_engine* engine, size_t batch, const double* u, const double* v,
                  const double* w, double* out, int median, void* stream);

/* Estimator path of the FCS / TS engines (iuv and uvw; the other backends
 * ignore it). ST_PATH_SPECTRAL: the reference's formulation, FFT correlation
 * against the cached spectra (shared-memory or cluster transforms).
 * ST_PATH_DIRECT: the same correlation in the time domain —
 * est[i] = s_f(i) sum_{i1} a'(i1) Q[h_f(i) + h_c1(i1)],
 * Q[k] = sum_{i2} b'(i2) sk[k + h_c2(i2)] (k < 2J - 1: no wrap at n = 3J - 2),
 * exact up to fp64 rounding, cost (2J - 1) I_c2 + I_f I_c1 multiply-adds per
 * item; hash lengths up to where Q fits one CTA's shared memory.
 * ST_PATH_AUTO (default): the direct path when its cost is below the
 * transforms' (engine.cu use_direct). Returns ST_EINVAL for an unknown path. */
enum { ST_PATH_AUTO = 0, ST_PATH_SPECTRAL = 1, ST_PATH_DIRECT = 2 };
int st_engine_set_path(st_engine* engine, int path);

/* T <- T - weight * u o v o w in sketch space (device vectors).
 * Replaces FcsEngine::deflate, cpd.cpp:79-87. */
int st_engine_deflate(st_engine* engine, double weight, const double* u, const double* v,
                      const double* w, void* stream);

/* HOST. Sketched robust tensor power method on a cubical device tensor:
 * FCS engine, num_inits restarts advanced in lockstep as one batch, strict-`>`
 * argmax, refinement, weight, deflation — cpd.cpp:234-277 with the same
 * initial-vector stream (SplitMix64(mix(seed ^ 0x7274706d)), random_unit
 * cpd.cpp:199-204). Outputs host weights[rank] and factor dim x rank
 * (column-major). Replaces rtpm(const DenseTensor&, const RtpmConfig&)
 * with backend FCS. */
int st_rtpm(int dtype, const void* tensor, size_t dim, size_t rank, size_t num_inits,
            size_t num_iters, size_t hash_len, size_t sketch_count, uint64_t seed,
            double* weights, double* factor, void* stream);
/* HOST. st_rtpm with RtpmConfig::backend (any ST_BACKEND_*). */
int st_rtpm_backend(int backend, int dtype, const void* tensor, size_t dim, size_t rank,
                    size_t num_inits, size_t num_iters, size_t hash_len, size_t sketch_count,
                    uint64_t seed, double* weights, double* factor, void* stream);

/* HOST. Alternating rank-1 power method for a general order-3 device tensor
 * (rtpm_asym, cpd.cpp:279-335): restarts batched in lockstep, each sweep
 * three engine iuv calls (free modes 0, 1, 2) with row normalisation, argmax
 * of |T(u,v,w)| (strict >), refinement, sign absorbed into the first factor,
 * deflation. Init stream SplitMix64(mix(seed ^ 0x72743161)). Outputs host
 * weights[rank] and factors packed as dims[0] x rank, dims[1] x rank,
 * dims[2] x rank (each column-major). */
int st_rtpm_asym(int backend, int dtype, const void* tensor, const size_t* dims, size_t rank,
                 size_t num_inits, size_t num_iters, size_t hash_len, size_t sketch_count,
                 uint64_t seed, double* weights, double* factors, void* stream);

/* HOST. Alternating least squares (als, cpd.cpp:337-383): MTTKRP columns from
 * one batched engine iuv per mode, exact Gram (F_o1^T F_o1 .* F_o2^T F_o2),
 * minimum-norm solve, column normalisation into the weights, and the device
 * residual_norm each sweep with the |prev - residual| < tol stop. Init stream
 * SplitMix64(mix(seed ^ 0x616c73)). Outputs as st_rtpm_asym; *sweeps (may be
 * NULL) receives the number of sweeps run. */
int st_als(int backend, int dtype, const void* tensor, const size_t* dims, size_t rank,
           size_t max_iters, double tol, size_t hash_len, size_t sketch_count, uint64_t seed,
           double* weights, double* factors, size_t* sweeps, void* stream);

/* || T - densify(cp) ||_F / || T ||_F (residual_norm, cpd.cpp:385-392) for an
 * order-3 device tensor and a device CP (weights[rank], factors packed as in
 * st_rtpm_asym). *out is a HOST double; 0 when both norms are 0, +inf when
 * only ||T|| is. */
int st_residual_norm(int dtype, const void* tensor, const size_t* dims, const double* weights,
                     size_t rank, const double* factors, double* out, void* stream);

/* densify(cp) (tensor.cpp:86-115): out (device, prod dims fp64, column-major)
 * = sum_r w_r u_r^(1) o ... o u_r^(N); factors: HOST array of device I_n x R
 * column-major matrices, weights device. */
int st_densify(size_t order, const size_t* dims, size_t rank, const double* weights,
               const double* const* factors, double* out, void* stream);

/* psnr(reference, estimate) (cpd.cpp:394-403): 10 log10(peak^2 / MSE) with
 * peak = max |reference|, capped at 99 dB (99 when MSE = 0); n elements of
 * two device tensors of the same dtype; *out HOST. */
int st_psnr(int dtype, const void* reference, const void* estimate, size_t n, double* out,
            void* stream);

/* ------------------------------------ inner products, regression, codecs */

/* Sketched inner product <a, b> of two device tensors of the same shape:
 * D families from families_for(dims, {hash_len, D, seed}); per family the dot
 * of the two sketches (kind ST_SKETCH_FCS: inner_once, estimators.cpp:193-196;
 * ST_SKETCH_TS: inner_once_ts, estimators.cpp:235-239), then median_reduce
 * (estimate_inner, estimators.cpp:198-207). estimates (device, D doubles) and
 * out (HOST, the median) may each be NULL. */
int st_estimate_inner(int kind, int dtype, const void* a, const void* b, size_t order,
                      const size_t* dims, size_t hash_len, size_t sketch_count, uint64_t seed,
                      double* estimates, double* out, void* stream);
/* out[k] = <a_k, b_k> for `count` device sketch rows of length len (fixed
 * summation order): the dot of inner_once / inner_once_ts for any family. */
int st_sketch_dots(size_t count, size_t len, const double* a, const double* b, double* out,
                   void* stream);

/* Sketched regression-layer forward map (Eq. 20):
 * Y[b][c] = median_d <FCS_d(X_b), FCS_d(W_c)> + bias[c], with X batch rows and
 * W classes rows, each row an order-`order` tensor of shape dims (column-major,
 * rows contiguous: x is batch x prod(dims), w is classes x prod(dims)). All
 * rows of one family are sketched by one K1 launch. bias (device) may be NULL;
 * y is device batch x classes. */
int st_regression_forward(int dtype, const void* x, size_t batch, const void* w, size_t classes,
                          const double* bias, size_t order, const size_t* dims, size_t hash_len,
                          size_t sketch_count, uint64_t seed, double* y, void* stream);

/* compress_contraction: FCS of A (x)_{3,1} B for device
 * tensors A (dims_a = I1, I2, L) and B (dims_b = L, I3, I4) without forming
 * the order-4 result: sum_l FCS(A(:,:,l); pairs 0,1) * FCS(B(l,:,:); pairs 2,3)
 * through the FFT. packed: D families of 4 pairs (I1, I2, I3, I4 entries,
 * st_family_tables layout); out D x (sum J_n - 3). L = 1 is compress_kron. */
int st_fcs_contraction(int dtype, const void* a, const size_t* dims_a, const void* b,
                       const size_t* dims_b, size_t sketch_count, const uint32_t* packed,
                       const size_t* hash_lens, double* out, void* stream);

/* decompress_kron / decompress_contraction:
 * out[q] = median_d prod_n s_n(i_n) * sketch_d[(sum_n h_n(i_n)) mod len] for
 * `count` device multi-indices idx (count x order, uint32), order <= 4. */
int st_sketch_decompress(const double* sketch, size_t sketch_count, size_t len,
                         const uint32_t* packed, size_t order, const size_t* dims, size_t count,
                         const uint32_t* idx, double* out, void* stream);
/* Full Kronecker reconstruction: out is the (I1 I3) x (I2 I4) column-major
 * estimate of A (x) B, row = I3 i1 + i3, col = I4 i2 + i4 (dims4 = I1..I4). */
int st_kron_decompress_all(const double* sketch, size_t sketch_count, size_t len,
                           const uint32_t* packed, const size_t* dims4, double* out, void* stream);

/* ------------------------------------------------------------ multi-GPU */
/* NCCL-aware entries for a C/C++ host that owns an NCCL communicator
 * (ncclComm_t passed as void*; NCCL is resolved at run time from
 * libnccl.so.2, so a process that already loaded NCCL shares it). One
 * process per GPU; the partitions are SURVEY.md §8(e)'s. Failures -> ST_ENCCL. */
size_t st_nccl_unique_id_bytes(void);                /* sizeof(ncclUniqueId) */
int st_nccl_get_unique_id(void* id);                 /* ncclGetUniqueId on rank 0 */
int st_nccl_comm_init_rank(void** comm, int nranks, const void* id, int rank);
int st_nccl_comm_destroy(void* comm);
/* HOST. The balanced contiguous share [lo, lo + count) of n items owned by
 * `rank` of `world` (the slab / rank-range rule of every sharded entry). */
int st_shard_range(size_t n, int rank, int world, size_t* lo, size_t* count);

/* Element-sharded dense FCS: `slab` (device) holds this rank's slab
 * i_{N-1} in st_shard_range(dims[N-1], rank, world) of the FULL tensor
 * `dims`; K1 sketches it into out (D x J~, device) and one ncclAllReduce
 * (sum, fp64) leaves the whole tensor's sketch on every rank. workspace as
 * st_fcs_dense_workspace(dtype, order, dims, count, D, hash_lens).
 * Replaces fcs_sketch(const DenseTensor&, const HashFamily&), sketch.cpp:187-201
 * (D families) for a tensor distributed over the communicator's GPUs. */
int st_fcs_dense_nccl(int dtype, const void* slab, size_t order, const size_t* dims,
                      size_t sketch_count, const uint32_t* packed, const size_t* hash_lens,
                      double* out, void* workspace, size_t workspace_bytes, void* comm,
                      void* stream);

/* Rank-sharded CP-form FCS: every rank holds the whole CP tensor (device),
 * sketches the CP ranks st_shard_range(rank, me, world) (frequency-domain
 * sum, st_fcs_cp) and one ncclAllReduce sums the D x J~ partials.
 * Replaces fcs_sketch(const CpTensor&, const HashFamily&), sketch.cpp:203-207. */
int st_fcs_cp_nccl(const double* weights, size_t rank, size_t order, const size_t* dims,
                   const double* const* factors, size_t sketch_count, const uint32_t* packed,
                   const size_t* hash_lens, double* out, void* workspace, size_t workspace_bytes,
                   void* comm, void* stream);

/* ---------------------------------------------------------- synthetic data */

/* HOST. n draws of SplitMix64(seed).next_gaussian() (rng.cpp:8-21), host libm,
 * multi-threaded through the counter identity; bit-identical to the serial
 * reference stream. */
int st_host_gaussian(uint64_t seed, size_t n, double* out, int threads);

/* Device fill of n iid N(0,1) values (SplitMix64 counter + Box-Muller, CUDA
 * libm: same distribution as the host stream, not bit-identical). For the
 * large benchmark tensor only. dtype ST_F32 / ST_F64. */
int st_device_gaussian(int dtype, uint64_t seed, size_t n, void* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FCS_B200_H */
