/*
 * ocsc_b200.h -- C-ABI of libocsc_b200.so, the B200 (sm_100a) hot path of
 * online convolutional sparse coding (arXiv 1706.06972).
 *
 * The reference (`ocsc`, pure Python/numpy) has no FFI; its boundary is the
 * Python API of pkg/src/ocsc/__init__.py.  Each entry point below replaces
 * the numpy arithmetic of one reference function (cited file:line, relative to
 * the reference's pkg/src/ocsc/).  The Python package paper_1706_06972_b200
 * binds these with ctypes and keeps the reference's
 * names, signatures and exceptions on top.
 *
 * Conventions
 *   - Every pointer is a DEVICE pointer owned by the caller unless noted;
 *     everything is enqueued on `stream` (a cudaStream_t, NULL = legacy
 *     default) and returns without a host sync unless noted.
 *   - dtype: OCSC_F32 (float / complex64) or OCSC_F64 (double / complex128).
 *     Complex arrays are interleaved (re, im) pairs.
 *   - Grids are H x W (a 1-D signal of length W is H = 1).  Half spectra
 *     ("rfft2 layout") are H x Wh with Wh = W/2 + 1, nfreq = H*Wh; planes are
 *     stored (plane, H, W) / (plane, H, Wh), row-major.
 *   - Forward transforms are unnormalised; inverse transforms carry 1/P
 *     (transforms.py:1-8).
 *   - Packed Hermitian matrices store the lower triangle row by row:
 *     entry (i, j), j <= i, at i*(i+1)/2 + j; one matrix per frequency.
 *   - Return value: OCSC_OK or a negative status; ocsc_last_error() gives
 *     the message of the last failure on the calling thread.
 */
#ifndef OCSC_B200_H
#define OCSC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OCSC_ABI_VERSION 1

#define OCSC_F32 4
#define OCSC_F64 8
#define OCSC_U8 1            /* image input only (ocsc_preprocess)          */

#define OCSC_OK 0
#define OCSC_ESHAPE (-1)    /* errors.py:4-5  ShapeMismatchError            */
#define OCSC_EDIVERGED (-2) /* errors.py:12-13 DivergenceError              */
#define OCSC_EUNINIT (-3)   /* errors.py:16-17 UninitializedHistoryError    */
#define OCSC_ECUDA (-4)     /* CUDA / cuFFT failure                         */
#define OCSC_EARG (-6)      /* bad dtype / unsupported size                 */

const char* ocsc_last_error(void);
int ocsc_abi_version(void);
/* Number of this library's own kernels enqueued so far in the process (cuFFT's excluded). */
int64_t ocsc_kernel_launches(void);

/* ------------------------------------------------------------ transforms --
 * transforms.py:82-87, 148-158 (forward_dft[_cols]); :90-109, 161-176
 * (inverse_dft[_cols] + the imaginary-residue guard). */

/* Create (and cache) the R2C and C2R plans for nplanes planes of H x W now, so the first
 * transform of that batch does not pay plan creation (OnlineTrainer's per-sample step path). */
int ocsc_fft_prepare(int dtype, int H, int W, int nplanes);
/* xh[n] = rfft2(x[n]) for n < nplanes; x (nplanes,H,W) real -> xh (nplanes,H,Wh). */
int ocsc_rfft2(int dtype, int H, int W, int nplanes, const void* x, void* xh, void* stream);
/* x[n] = irfft2(xh[n]) / P.  xh is CLOBBERED (cuFFT C2R). */
int ocsc_irfft2(int dtype, int H, int W, int nplanes, void* xh, void* x, void* stream);
/* Full complex DFT of reference columns (P, ncols), K fastest, row-major (H, W) pixels.
 * in_complex = 0: `in` is real (P, ncols); 1: complex.  inverse = 1 uses e^{+i}; no scaling. */
int ocsc_dft_cols(int dtype, int H, int W, int ncols, const void* in, int in_complex, void* out,
                  int inverse, void* stream);
/* stats[0] = max |Im spatial|, stats[1] = max |spec| over n complex entries each
 * (atomic max; caller zeroes stats).  transforms.py:102-109 */
int ocsc_residue_stats(int dtype, int64_t n, const void* spatial, const void* spec, double* stats,
                       void* stream);
/* out[i] = scale * Re(in[i]) */
int ocsc_real_part(int dtype, int64_t n, const void* in, double scale, void* out, void* stream);
/* half spectra (nplanes, H, Wh) -> full spectrum columns (P, nplanes) by Hermitian extension */
int ocsc_half_to_cols(int dtype, int H, int W, int nplanes, const void* half, void* cols, void* stream);
/* full spectrum columns (P, ncols) -> half spectra (ncols, H, Wh) (gather) */
int ocsc_cols_to_half(int dtype, int H, int W, int ncols, const void* cols, void* half, void* stream);
/* stats[0] = max |X[p] - conj X[-p]|, stats[1] = max |X| over columns (P, ncols) (caller zeroes) */
int ocsc_hermitian_defect(int dtype, int H, int W, int ncols, const void* cols, double* stats,
                          void* stream);

/* ---------------------------------------------------------------- coding --
 * coding.py:45-134 */

/* coding.py:45-48 */
int ocsc_soft_threshold(int dtype, int64_t n, const void* in, double kappa, void* out, void* stream);
/* coding.py:51-64, rows (nrows, K) complex, x (nrows) complex */
int ocsc_solve_code_rows(int dtype, int nrows, int K, const void* d, const void* x, const void* t,
                         double rho, void* out, void* stream);
/* den[p] = rho + sum_k |Wh[k][p]|^2, Wh (K, nfreq) */
int ocsc_code_den(int dtype, int K, int nfreq, const void* Wh, double rho, void* den, void* stream);
/* Bytes of scratch ocsc_code_admm needs for (H, W, K, B); want_z adds the z buffer. */
size_t ocsc_code_workspace_bytes(int dtype, int H, int W, int K, int B, int want_z);
/* Batched ADMM sparse coding, coding.py:67-119, for B samples against one dictionary.
 *   xh   (B, nfreq)       sample spectra (ocsc_rfft2 of the samples)
 *   Wh   (K, nfreq)       dictionary spectrum;  den (nfreq) from ocsc_code_den
 *   u, t (B, K, H, W)     in: code U and U - Gamma (zeros = cold start); out: final values
 *   zh   (B, K, nfreq)    optional (NULL): spectrum of the last ADMM iterate z
 *   iters, status (B)     int32: iterations run; 0 = hit max_iters, 1 = converged,
 *                         2 = diverged (non-finite code) at iteration iters[b]
 * Each sample stops at exactly the iteration the reference would (the
 * two-part test of coding.py:113-118); converged samples are frozen on device.
 * poll > 0: the host checks the all-converged flag every `poll` iterations,
 * one chunk behind the device (no pipeline bubble); poll = 0 never syncs. */
int ocsc_code_admm(int dtype, int H, int W, int K, int B, const void* xh, const void* Wh,
                   const void* den, double beta, double rho, int max_iters, double rel_tol,
                   void* u, void* t, void* zh, void* work, int32_t* iters, int32_t* status,
                   int poll, void* stream);
/* Fused on-chip code ADMM (cold start) + objective for grids with an instantiated
 * kernel: one thread-block cluster per sample keeps the ADMM state in shared memory
 * for every iteration; the cluster exchanges the partial synthesis through DSMEM.
 * Outputs u (B,K,H,W) = code U, t (optional) = U - Gamma, uh (B,K,nfreq) = rfft2(U),
 * obj/resid as ocsc_code_objective, iters/status as ocsc_code_admm.  Same
 * stopping semantics as ocsc_code_admm.  ocsc_code_fused_cluster returns the cluster
 * size the launch would use, or 0 when (dtype, H, W, K) is not supported. */
int ocsc_code_fused_cluster(int dtype, int H, int W, int K, int B);
/* Launch plan of ocsc_code_fused (host array of 8 int32): main cluster size, threads per
 * CTA, dynamic shared memory bytes, registers per thread, main-shape resident clusters,
 * b_split = samples the plan finishes before its last main round starts (B when it has
 * one round), then the cluster size and resident clusters of the plan for the remaining
 * B - b_split samples (0, 0 when b_split = B): a caller that splits the batch there can
 * overlap work with the second part.  Returns the main cluster size (0 = unsupported). */
int ocsc_code_fused_info(int dtype, int H, int W, int K, int B, int32_t* info);
/* Concurrent-plan details of ocsc_code_fused (host array of 8 int32): side cluster size
 * (0 = the plan is sequential: main waves + optional tail), side clusters launched, side
 * shape keeps D in registers, main clusters launched (persistent), samples per schedule
 * row, main shape keeps D in registers, modelled makespan x 1000, concurrent flag.  A
 * concurrent plan runs the main shape persistent and a narrower side shape on the SMs the
 * main clusters leave free, launched programmatically behind it on the same stream. */
int ocsc_code_fused_side_info(int dtype, int H, int W, int K, int B, int32_t* info);
/* Development aid: device buffer of 64 int64 that receives clock64() phase stamps of CTA 0
 * for iterations 8..15 of the next fused launches (NULL disables). */
int ocsc_debug_fused_profile(void* buf);
int ocsc_debug_chol_profile(void* buf);  /* dev aid: clock64 phase stamps of the blocked Cholesky (CTA 0) */
int ocsc_debug_plane_profile(void* buf);   /* debug: clock64 phase stamps of the plane-resident stream kernel */
/* Development aid: device buffer of 2*B int64 receiving %globaltimer at each sample's start/end. */
int ocsc_debug_fused_timeline(void* buf);
/* Development aid: device buffer of 1024 int64: %globaltimer (first 512) and clock64 (last 512)
 * at the start of each of the first 512 iterations of CTA 0 of the next fused launches. */
int ocsc_debug_fused_iterations(void* buf);
int ocsc_code_fused(int dtype, int H, int W, int K, int B, const void* xh, const void* Wh,
                    const void* den, double beta, double rho, int max_iters, double rel_tol,
                    void* u, void* t, void* uh, double* obj, double* resid, int32_t* iters,
                    int32_t* status, void* stream);
/* Streaming code ADMM (coding.py:67-119, cold start) for grids whose state does not fit on
 * chip: the same single-state iteration as ocsc_code_fused with w in `u` (HBM) and
 * hand-written Good-Thomas row/column FFT passes (100 x 100 and 266 x 266: BASELINE configs
 * 0, 2, 3).  On return u holds the codes U = S(w); iters/status as ocsc_code_admm.  `work`
 * holds ocsc_code_stream_workspace_bytes() bytes. */
int ocsc_code_stream_supported(int dtype, int H, int W);
/* CTAs (one per SM) one code iteration of the plane-resident streaming kernel occupies for this
 * batch (float32 100 x 100), 0 when another path runs; the rest of the SMs are free for overlap. */
int ocsc_code_stream_plane_ctas(int dtype, int H, int W, int K, int B);
size_t ocsc_code_stream_workspace_bytes(int dtype, int H, int W, int K, int B);
int ocsc_code_stream(int dtype, int H, int W, int K, int B, const void* xh, const void* Wh, const void* den,
                     double beta, double rho, int max_iters, double rel_tol, void* u, void* work,
                     int32_t* iters, int32_t* status, int poll, void* stream);
/* coding.py:122-134 for B codes: uh = rfft2(u) (B, K, nfreq) and
 * obj[b] = 0.5 ||x_b - sum_k w_k (*) u_bk||^2 + beta ||u_b||_1 (double, device);
 * resid[b] (optional) = ||x_b - reconstruction||^2 (evaluate.py:55-62 PSNR input). */
int ocsc_code_objective(int dtype, int H, int W, int K, int B, const void* xh, const void* Wh,
                        const void* u, double beta, void* uh, double* obj, double* resid,
                        void* stream);
/* out[b][p] = sum_k Wh[k][p] zh[b][k][p]  (reconstruct, coding.py:122-126, in frequency) */
int ocsc_synthesize(int dtype, int K, int nfreq, int B, const void* Wh, const void* zh, void* out,
                    void* stream);

/* --------------------------------------------------------------- history --
 * dictionary.py:30-131.  State is kept as SUMS: S_p = sum z z^H (packed),
 * c_p = sum conj(x) z, with the count t on the host; the reference's averaged
 * cross = c/t and inv_gram = t (S + t rho P I)^-1 are the same quantities. */

/* S (nfreq, K(K+1)/2), c (nfreq, K) += rank-B update; z element (b,k,p) at
 * z[b*z_sb + k*z_sk + p*z_sp], x element (b,p) at x[b*x_sb + p*x_sp]. */
int ocsc_history_accumulate(int dtype_in, int dtype_hist, int K, int nfreq, int B, const void* z,
                            int64_t z_sb, int64_t z_sk, int64_t z_sp, const void* x, int64_t x_sb,
                            int64_t x_sp, void* S, void* c, void* stream);
/* inv_p = scale * (S_p + ridge I)^-1, per-frequency in-place Gauss-Jordan (HPD, no pivoting)
 * in registers/shared memory, computed in dtype_hist and stored packed as dtype_inv
 * (complex64 storage for float32 training halves the bytes the J row solves re-read).
 * K <= 118 (complex128) / 167 (complex64).
 * info (device int32): 0, or 1 + a frequency whose matrix was not positive definite. */
int ocsc_history_invert(int dtype_hist, int dtype_inv, int K, int nfreq, const void* S, double ridge,
                        double scale, void* inv, int32_t* info, void* stream);
/* Persistent form of ocsc_history_invert (32 < K <= 100): `ctas` CTAs claim frequencies from the
 * device counter *ctr (zeroed by the caller) until none are left, so a few CTAs can run beside
 * another kernel and a later full-grid launch sharing the counter finishes the rest.  info is
 * not reset. */
int ocsc_history_invert_claim(int dtype_hist, int dtype_inv, int K, int nfreq, const void* S, double ridge,
                              double scale, void* inv, int32_t* info, int32_t* ctr, int ctas, void* stream);
/* Low-rank refresh of a packed inverse (Woodbury): out_p = (A_p + U_p U_p^H)^-1 from
 * inv_in_p = A_p^-1 (packed complex128, e.g. ocsc_history_invert with dtype_inv = f64), U_p the
 * K x nb code spectra z element (b,k,p) at z[b*z_sb + k*z_sk + p*z_sp], nb <= 16; out packed as
 * dtype_out.  Lets a trainer invert S plus most of a mini-batch while the rest is still being
 * coded, then fold the remainder in O(K^2 nb) (no reference counterpart; same result as
 * ocsc_history_invert of the full sum).  info as ocsc_history_invert (capacitance matrix).
 * With S, c non-NULL (complex128 history sums) the same nb samples are folded into them in the
 * same pass (x element (b,p) at x[b*x_sb + p*x_sp], dtype_z), as ocsc_history_accumulate would. */
int ocsc_history_woodbury(int dtype_z, int dtype_out, int K, int nfreq, int nb, const void* inv_in,
                          const void* z, int64_t z_sb, int64_t z_sk, int64_t z_sp, void* out,
                          int32_t* info, const void* x, int64_t x_sb, int64_t x_sp, void* S, void* c,
                          void* stream);
size_t ocsc_history_woodbury_smem(int K, int nb);
/* Large K (BASELINE configs 3-4; any K): blocked right-looking Cholesky of S_p + ridge I per
 * frequency (one CTA per frequency, 32x32 tiles, panel staged in shared memory).  L is written
 * full (nfreq, Kp, Kp), lower triangle, Kp = K rounded up to a multiple of 32 (the padding is
 * the decoupled block ridge * I, so rows/columns >= K never touch the history's solution);
 * ocsc_history_factor_bytes gives its size.  info as ocsc_history_invert. */
size_t ocsc_history_factor_bytes(int dtype_hist, int K, int nfreq);
int ocsc_history_factor(int dtype_hist, int K, int nfreq, const void* S, double ridge, void* L,
                        int32_t* info, void* stream);
/* packed (nfreq, K(K+1)/2) Hermitian -> full (nfreq, K, K), times scale */
int ocsc_packed_to_full(int dtype, int K, int nfreq, const void* packed, double scale, void* full,
                        void* stream);
/* flag (device int32) |= 1 if any of n values (complex: 2n reals) is non-finite */
int ocsc_nonfinite(int dtype, int64_t n_reals, const void* a, int32_t* flag, void* stream);

/* ------------------------------------------------------------ dictionary --
 * dictionary.py:134-215 */

/* Row solve, dictionary.py:134-142, in sum form:
 * conj(D_p) = inv_p (c_p + ridge conj(V_p - Theta_p)), inv from ocsc_history_invert
 * with scale 1, ridge = t rho P.  V/Theta/D element (k,p) at [k*sk + p*sp]. */
int ocsc_dict_rowsolve(int dtype, int dtype_hist, int dtype_inv, int K, int nfreq, const void* inv,
                       const void* c, double ridge, const void* Vh, const void* Th, int64_t sk, int64_t sp,
                       void* Dh, void* stream);
/* Row solve with the Cholesky factor of ocsc_history_factor (two triangular solves per
 * frequency): conj(D_p) = L^-H L^-1 (c_p + ridge conj(V_p - Theta_p)).  K is the history's
 * order (L padded as ocsc_history_factor writes it). */
int ocsc_dict_rowsolve_chol(int dtype, int dtype_hist, int K, int nfreq, const void* L, const void* c,
                            double ridge, const void* Vh, const void* Th, int64_t sk, int64_t sp,
                            void* Dh, void* stream);
/* One fused projection round on half spectra (K, H, Wh), dictionary.py:145-154 + :205-207:
 * alpha_k = crop(irfft2(D_k + Theta_k)) / max(||.||, 1); V_k = rfft2(pad(alpha_k));
 * Theta_k += D_k - V_k.  Pruned separable DFTs: only the M0 x M1 support is touched.
 * alpha (K, M0*M1) row-major support. */
int ocsc_dict_project(int dtype, int H, int W, int M0, int M1, int K, const void* Dh, void* Th,
                      void* Vh, void* alpha, void* stream);
/* alpha_k = crop(irfft2(X_k)) without normalisation (training.py:165-169 final_filters). */
int ocsc_crop_irfft(int dtype, int H, int W, int M0, int M1, int K, const void* Xh, void* alpha,
                    void* stream);
/* Full-spectrum projection tail on reference columns: spatial (P, K) real ->
 * padded (P, K) real with the support scaled into the unit ball. */
int ocsc_crop_normalize_cols(int dtype, int H, int W, int M0, int M1, int K, const void* spatial,
                             void* padded, void* stream);
/* Support (K, M0*M1) -> spectra (K, H, Wh) via the pruned forward DFT (dict_state_from_filters). */
int ocsc_support_rfft(int dtype, int H, int W, int M0, int M1, int K, const void* alpha, void* Vh,
                      void* stream);
/* Frequency-sharded projection (SURVEY.md 8(e) exchange B).  A rank owns rows [u0, u1) of
 * the (H, Wh) half plane; slice arrays are (K, u1-u0, Wh).
 * ocsc_crop_irfft_rows: apart (K, M0*M1) float64 = this slice's share of
 *   crop(irfft2(X + Theta)) (Theta may be NULL); summed over all slices (an all-reduce) it is
 *   the full crop of dictionary.py:149.
 * ocsc_normalize_support: alpha = apart / max(||apart_k||, 1) (dictionary.py:150-152).
 * ocsc_support_rfft_rows: V = rfft2(pad(alpha)) on the slice rows; with D and Theta given also
 *   Theta += D - V there (dictionary.py:153-154, 205-207). */
int ocsc_crop_irfft_rows(int dtype, int H, int W, int M0, int M1, int K, int u0, int u1, const void* Xh,
                         const void* Th, double* apart, void* stream);
int ocsc_normalize_support(int dtype, int M, int K, const double* apart, void* alpha, void* stream);
int ocsc_support_rfft_rows(int dtype, int H, int W, int M0, int M1, int K, int u0, int u1, const void* alpha,
                           void* Vh, const void* Dh, void* Th, void* stream);
/* Tolerance test of the batch dictionary update (dictionary.py:210-214): per filter k,
 * out[2k] = ||D_k - V_k||^2, out[2k+1] = ||D_k||^2 over the full spectrum, from half spectra
 * (K, H, Wh) with Hermitian weights. */
int ocsc_dict_gaps(int dtype, int H, int W, int K, const void* Dh, const void* Vh, double* out, void* stream);
/* out[0] += sum (a-b)^2, out[1] += sum a^2 over n reals (b may be NULL: treated as 0) */
int ocsc_norms2(int dtype, int64_t n, const void* a, const void* b, double* out, void* stream);

/* Image preparation (preprocessing.py:36-100), ONE kernel over N images of H x W (channels 1,
 * or 3 interleaved RGB mixed with the luminance weights :13).  flags bit 0: local contrast
 * normalisation, Gaussian window `lcn_window` / `lcn_sigma`, std floor `lcn_epsilon` (:58-71);
 * bit 1: edge taper with kernel size = ramp width `taper_size` (:74-89) and per-image width
 * taper_sigmas[i] (device pointer), or, when taper_sigmas is NULL, numpy's
 * default_rng(taper_seed0 + i).uniform(lo, hi) drawn on the device (:98-99, cli.py:116).
 * scipy "reflect" borders; float64 arithmetic.  dtype_in: OCSC_U8 / OCSC_F32 / OCSC_F64;
 * dtype_out: OCSC_F32 / OCSC_F64.  Replaces preprocess() per image (preprocessing.py:92). */
int ocsc_preprocess(int dtype_in, int dtype_out, int N, int H, int W, int channels, const void* in, int flags,
                    int lcn_window, double lcn_sigma, double lcn_epsilon, int taper_size,
                    const double* taper_sigmas, int64_t taper_seed0, double taper_sigma_lo,
                    double taper_sigma_hi, void* out, void* stream);
/* Host-side: out[i] = numpy default_rng(seed0 + i).uniform(lo, hi) (SeedSequence + PCG64),
 * bit-identical to numpy 2.x; the taper widths ocsc_preprocess draws (preprocessing.py:98-99). */
int ocsc_taper_sigmas(int64_t seed0, int n, double lo, double hi, double* out);

#ifdef __cplusplus
}
#endif
#endif /* OCSC_B200_H */
