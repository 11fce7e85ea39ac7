/* mps_b200.h — C ABI of the B200-native multiprecision MPS gate update.
 *
 * What this library computes (citations: P:L = /root/reference/PAPER.md line L,
 * S:L = SPEC.md line L; the full reading list is in DESIGN.md):
 *   The state |Psi> of n qubits is held in the matrix-product form of Eq. 1
 *   (P:240-247): site tensors Q_s(i_s, v_{s-1}, v_s) with 2 x m_{s-1} x m_s
 *   elements (Vidal's Gamma) and bond vectors V_s(v_s) of Schmidt
 *   coefficients (Eq. 2; Vidal's lambda).  A U(4) gate on
 *   qubits (s, s+1) updates only Q_s, V_s, Q_{s+1} by
 *     Theta = U . (lambda_{s-1} Gamma_s lambda_s Gamma_{s+1} lambda_{s+1}),
 *     one-sided Jacobi SVD of Theta reshaped (2 chi_l) x (2 chi_r),
 *     truncation of small Schmidt coefficients and to chi_max,
 *     renormalisation of the kept coefficients, split back into Gamma_s, Gamma_{s+1}
 *   (BASELINE.json north_star).  U(8) gates on three
 *   adjacent qubits are elementary (three-site update, right
 *   site split first); a two-qubit gate on (s, s+2) is embedded into U(8)
 *   (S:336); U(2) gates update one site.
 *   All arithmetic is multiprecision complex floating point with >= p
 *   significant bits and a 64-bit exponent (BASELINE north_star; precision knob
 *   zkcm_set_default_prec).  Supported p: 64 <= p <= 512.
 *
 * Number interchange format (host buffers; one "record" per real):
 *     int64_t exp; uint32_t sign; uint32_t reserved; uint32_t limb[L];  L = ceil(p/32)
 *     value = (-1)^sign * (sum_k limb[k] 2^(32k)) * 2^(exp - 32L)
 *     nonzero: limb[L-1] >= 2^31 and the low 32L-p bits are zero (exactly p bits);
 *     zero: all limbs 0 and exp = INT64_MIN.       sizeof = mps_record_bytes(p).
 *   A complex number is its re record followed by its im record.
 *   A site tensor is row-major [i][a][b] (i physical, a left bond, b right bond).
 *   A gate U on k qubits is a row-major 2^k x 2^k complex matrix; basis index
 *   x = sum_t i_t 2^(k-1-t) with the first listed qubit most significant
 *   (qubit 0 = MSB; matches the |000> labels of P:351).
 *
 * Ownership: every pointer argument is borrowed for the duration of the call
 * only; inputs are copied, never modified.  Output buffers are caller
 * allocated host memory (sizes stated per call).  Device memory is owned by the
 * library.  A handle is used by one host thread at a time.
 *
 * Errors: functions return MPS_OK (0) or a negative status.  Argument errors
 * return immediately without side effects.  Device-side failures (Jacobi
 * non-convergence, zero bond, CUDA errors) are sticky: the handle then only
 * accepts mps_free / mps_strerror and every other call returns the error.
 */
#ifndef MPS_B200_H
#define MPS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  MPS_OK = 0,
  MPS_EINVAL = -1,       /* bad argument: n < 1, chi_max < 1, bad sites, span > 3 */
  MPS_ENOTUNITARY = -2,  /* ||U^H U - I||_max > 2^(-p+16) */
  MPS_ENOCONV = -3,      /* Jacobi exceeded 60 sweeps (sticky) */
  MPS_EZEROBOND = -4,    /* no singular value above the truncation floor (sticky) */
  MPS_EOVERLAP = -5,     /* gates of one layer overlap */
  MPS_EUNSUPPORTED = -6, /* precision outside 64..512, chi beyond the compiled limits */
  MPS_ENOMEM = -7,
  MPS_ECUDA = -8,        /* CUDA runtime error (sticky); also: no CUDA device (the library never falls back to the CPU) */
  MPS_ENCCL = -9,
  MPS_ETOOBIG = -10      /* to_dense with n > 24 */
};

typedef struct mps_state mps_state; /* opaque */

size_t mps_record_bytes(int prec_bits);
const char* mps_strerror(int status);
/* Largest supported bond dimension chi_max (Theta up to 2chi x 2chi; 4chi rows for U(8)). */
int mps_max_chi(void);

/* ---- state lifecycle ------------------------------------------------------ */
/* Create |0...0> on the current CUDA device (all m_s = 1, V_s = [1]).
 *   n_qubits >= 1, 64 <= prec_bits <= 512, 1 <= chi_max <= mps_max_chi().
 *   trunc_thr: Schmidt coefficients sigma_j < trunc_thr * ||sigma||_2 are dropped
 *   (reading R4); <= 0 selects 2^-ceil(p/2).
 *   The threshold is taken exactly as the given binary64 value. */
int mps_init(mps_state** out, int n_qubits, int prec_bits, int chi_max, double trunc_thr);
void mps_free(mps_state* st); /* NULL-safe */
/* Run all subsequent work of this handle on the given cudaStream_t (NULL = legacy default). */
int mps_set_stream(mps_state* st, void* cuda_stream);

/* ---- gates ------------------------------------------------------------------ */
/* Apply U (2^k x 2^k complex records, host) on the k = 1..3 distinct qubits sites[0..k)
 * in any order and at any distance (the paper's applyU on chosen qubits, §3.2;
 * the n factor of O(g n m^3)).  sites[0] is the most significant bit of U's
 * row/column index.  Placement (R18): U is rewritten on ascending sites; (s, s+1)
 * and (s, s+1, s+2) are applied directly, (s, s+2) is embedded into U(8) with identity on
 * s+1; any other placement is routed with exact SWAP gates (each a two-site update,
 * truncating like any other) that bring the far qubits next to the lowest one and are
 * undone afterwards.  Validates unitarity at p bits.  MPS_EINVAL: k out of range, a site
 * out of range or repeated.  Synchronous w.r.t. the handle's stream. */
int mps_apply_gate(mps_state* st, const void* U, const int* sites, int k);
/* A layer of gates whose site spans [min, max] are pairwise disjoint (MPS_EOVERLAP
 * otherwise).  Adjacent two-site gates in ascending order run as batched launches; the
 * others one by one as mps_apply_gate.  U[g] points to gate g's records; sites_flat holds
 * the k[g] sites of each gate in order. */
int mps_apply_layer(mps_state* st, int n_gates, const void* const* U, const int* sites_flat, const int* k);

/* ---- queries (synchronise; results on the host) ------------------------------ */
/* c(b) = Gamma_0^{b0} lambda_0 Gamma_1^{b1} ... Gamma_{n-1}^{b_{n-1}} (Eq. 1, unnormalised). out: 1 complex. */
int mps_amplitude(mps_state* st, const uint8_t* bits, void* out);
/* <Psi|O|Psi> / <Psi|Psi> for O on contiguous ascending sites (k = 1..3). out: 1 complex. */
int mps_expect(mps_state* st, const void* O, const int* sites, int k, void* out);
/* Reduced density operator of k ascending sites (k <= 6), the paper's RDO_block(a,b) /
 * RDO(list): rho(x, x') = sum_rest psi(x, rest) conj(psi(x', rest)) / trace,
 * computed by transfer contraction (no 2^n state).  out: 2^k x 2^k complex, row-major,
 * x = first listed site most significant (the |000> labels of P:351). */
int mps_rdo(mps_state* st, const int* sites, int k, void* out);
/* <Psi|Psi> of the stored tensors. out: 1 real. */
int mps_norm2(mps_state* st, void* out);
/* All 2^n amplitudes, qubit 0 = MSB (n <= 24). out: 2^n complex. */
int mps_to_dense(mps_state* st, void* out);
int mps_sync(mps_state* st); /* first sticky error or MPS_OK */

/* ---- site-sharded blocks -----------------------------------------
 * A block state holds the global sites [site_lo, site_hi) of an n_total-site chain (one
 * block per GPU, contiguous).  The bonds site_lo-1 and site_hi-1 are external: their
 * Schmidt vectors are mirrored in both neighbouring blocks.  Gates fully inside a block use
 * mps_apply_gate / mps_apply_layer with LOCAL site indices.  A two-site gate on the block
 * edge (site_hi-1, site_hi) runs on the left block: the right block exports its first site
 * and the Schmidt vector right of it (device buffers), the left block applies the update and
 * returns the new first site of the right block and the new shared Schmidt vector, which the
 * right block imports.  The halo buffers move between GPUs by NCCL send/recv (the Python
 * driver, paper_1111_3124_b200/dist.py).  Device pointers below are CUDA device memory. */
int mps_init_block(mps_state** out, int n_total, int site_lo, int site_hi, int prec_bits, int chi_max,
                   double trunc_thr);
int mps_block_dims(mps_state* st, int* site_lo, int* n_local, int* m_ext_l, int* m_ext_r);
/* first local site [2][m_l][m_r] -> dG (device), Schmidt vector right of it (m_r reals) -> dlam (device, may be NULL) */
int mps_block_export_first(mps_state* st, void* dG, void* dlam, int* m_l, int* m_r);
/* U (host 4x4 records) on (last local site, halo site); dG_halo [2][m_ext_r][m_h] (device), dlam_h the
 * Schmidt vector right of the halo site (device, NULL at the chain end).  Outputs (device): the halo
 * site [2][k][m_h] and the new shared Schmidt vector (k reals); k_out host int. */
int mps_block_boundary_apply(mps_state* st, const void* U, const void* dG_halo, int m_h, const void* dlam_h,
                             void* dG_halo_out, void* dlam_mid_out, int* k_out);
/* replace the first local site by dG0 [2][k][m_r] and the external left Schmidt vector by dlam_mid (k) */
int mps_block_import_first(mps_state* st, const void* dG0, const void* dlam_mid, int k);
/* amplitude chain over the block: v_out = (v_in lambda_ext_l) Gamma_lo^{b0} lambda ... Gamma_hi-1^{b};
 * v_in: m_ext_l complex (host; ignored for the first block), v_out: m_ext_r complex (host; the
 * amplitude itself for the last block). bits: n_local entries. */
int mps_amplitude_block(mps_state* st, const uint8_t* bits, const void* v_in, void* v_out);

/* ---- diagnostics / test surface ----------------------------------------------- */
int mps_n_qubits(mps_state* st);
int mps_bond_dims(mps_state* st, int* out /* n-1 ints */);
/* Site tensor Gamma_site ([2][m_l][m_r] complex records) and Schmidt vector of a bond
 * (m reals).  The buffers may be HOST or DEVICE memory (unified addressing picks the
 * copy direction); the copy is ordered on the state's stream and complete on return.  The
 * site-sharded SPMD driver (paper_1111_3124_b200/dist.py) moves tensors between
 * ranks through device buffers with these four calls.  EINVAL: bad index, dims that differ
 * from the current bond dims (set_site), m outside [1, capacity of the bond] (set_schmidt). */
int mps_schmidt(mps_state* st, int bond, void* out /* m reals, may be NULL */, int* m);
int mps_get_site(mps_state* st, int site, void* out /* 2*m_l*m_r complex, may be NULL */, int* m_l, int* m_r);
/* set_schmidt may change the bond dimension; the caller then sets both neighbouring sites. */
int mps_set_schmidt(mps_state* st, int bond, const void* in, int m);
int mps_set_site(mps_state* st, int site, const void* in, int m_l, int m_r);
/* JSON: gates, sweeps_total, rotations, last gate sweeps, bond dims. */
int mps_stats(mps_state* st, char* json, size_t cap);

/* ---- kernel-level batch entry (BASELINE configs[1]; no MPS state) ---------------
 * For each item b < batch: Gamma_A, Gamma_B in C^{2 x chi x chi} ([i][a][b] records),
 * lambda_l, lambda_m, lambda_r (chi reals each, or NULL = all ones), U (4x4 complex).
 * Computes Theta' = U (lambda_l Gamma_A lambda_m Gamma_B lambda_r), its one-sided Jacobi
 * SVD, truncation to k <= chi_max with renormalisation and the split.
 * Outputs (host, caller allocated; any may be NULL):
 *   sigma   batch * 2chi reals: all singular values, descending
 *   k_out   batch ints
 *   A_out   batch * 2*chi*chi_max complex: Gamma_A' [i][a][b<k] with row stride chi_max
 *   B_out   batch * 2*chi_max*chi complex: Gamma_B' [j][b<k][c]
 *   lam_out batch * chi_max reals
 *   sweeps  batch ints (Jacobi sweeps, the final check-only sweep included)
 *   theta_debug: NULL, or batch*(2chi)^2 complex: Theta' column-major; when given,
 *                the call stops after the contraction (slice test).
 * Host<->device copies are part of the call (pinned host buffers make them DMA-speed).  Batches
 * of more than 592 items are processed in chunks of 592 items (four waves of the one-CTA-per-SM
 * kernels): the copies of one chunk run on two internal streams while another chunk computes on
 * cuda_stream; every item's result is independent of the chunking.  The device buffers come
 * from a grow-only arena kept between calls (calls are serialised).  The call returns after all
 * copies have completed. */
int mps_bench_update_batch(int prec_bits, int chi, int chi_max, int batch, double trunc_thr,
                           const void* A, const void* B, const void* lam_l, const void* lam_m,
                           const void* lam_r, const void* U, void* sigma, int* k_out, void* A_out,
                           void* B_out, void* lam_out, int* sweeps, void* theta_debug,
                           void* cuda_stream);

/* Same computation on DEVICE buffers (records, same layouts), no host copies, asynchronous
 * on cuda_stream (the measured kernel path of bench.py).  ws: device workspace of
 * mps_update_batch_workspace(prec_bits, chi, batch) bytes. */
size_t mps_update_batch_workspace(int prec_bits, int chi, int batch);
int mps_update_batch_device(int prec_bits, int chi, int chi_max, int batch, double trunc_thr,
                            const void* dA, const void* dB, const void* dlam_l, const void* dlam_m,
                            const void* dlam_r, const void* dU, void* dsigma, int* dk_out,
                            void* dA_out, void* dB_out, void* dlam_out, int* dsweeps, void* dws,
                            void* cuda_stream);
/* Number of kernel launches issued by the last mps_update_batch_device / bench call. */
int mps_last_launch_count(void);

/* ---- measurement: CUDA events around the kernel classes of the batch path, on the
 * launching stream.  which: 0 p-bit Jacobi SVD kernel (a3), 1 contraction+gate (a1-a2),
 * 2 truncate+split (a4-a5), 3 binary64 preconditioner + Newton-Schulz + refinement sweeps +
 * A_1 = Theta' X + first-order finish (R19, R22, R23), 4 recovery of V (R16); inside
 * those: 5 the binary64 phase of the block Jacobi, 6 the refinement-sweep kernels, 7 every
 * tensor-core MMA kernel, 8 the binary32 phase of the block Jacobi and its hand-over (R27).
 * enable(1) clears and starts recording; query syncs and sums the durations. */
int mps_profile_enable(int on);
int mps_profile_query(int which, double* total_ms, int* launches);
/* Totals over the Jacobi problems run since mps_profile_enable(1): [0] rotations applied,
 * [1] pair evaluations (gamma computed), [2] sum (sweeps+1) M N (norm passes),
 * [3] sum N N M (recovery of V), [4] digit products executed by the rotation phase
 * (zero-digit variants counted exactly), [5] Jacobi problems that ended on the certified
 * stop instead of a rotation-free sweep (R21), [6] algorithmic DFMA of the binary64
 * block Jacobi (Gram, inner rotations, W applications as formed), [7] int8 multiply-accumulates
 * issued to the tensor cores (MMAs x 128 x 128 x 32), [8] algorithmic FFMA of the binary32 phase
 * of the block Jacobi.  mps_profile_counts returns [0..3],
 * mps_profile_counts_n the first n (1..16; the rest reserved, 0).  bench.py derives the
 * roofline fractions from them. */
int mps_profile_counts(long long* out4);
int mps_profile_counts_n(long long* out, int n);

/* ---- kernel test surface --------------------------------------------------------
 * One-sided Jacobi SVD (a3) of `batch` column-major M x N complex matrices (host
 * records), sigma: batch*min(M,N) reals descending; sweeps: batch ints (may be NULL);
 * rot_per_sweep: batch*64 ints, rotations executed in sweep s (may be NULL). */
int mps_svd_batch(int prec_bits, int M, int N, int batch, const void* A, void* sigma, int* sweeps,
                  int* rot_per_sweep);
/* Elementwise device scalar arithmetic on n records (a, b, out host): op 0 a+b, 1 a-b,
 * 2 a*b, 3 a/b, 4 sqrt a, 5 1/sqrt a, 6 1/a, 7 copy, 8 round trip through the fixed-point
 * digit format.  Results are faithful (not correctly rounded) at p bits. */
int mps_debug_mpf(int prec_bits, int op, int n, const void* a, const void* b, void* out);

#ifdef __cplusplus
}
#endif
#endif /* MPS_B200_H */
