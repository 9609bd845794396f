/*
 * dilithium_b200.h -- C ABI of the B200-native batched CRYSTALS-Dilithium (round-3) engine.
 *
 * This is the drop-in boundary for the reference's batched hot path.  Each entry point
 * names the reference interface it replaces (paths relative to the reference's
 * proj/include/dilithium/).  Plain pointers and sizes only; the library owns device
 * memory, pinned staging and streams.  All batch calls are synchronous at the API and
 * internally asynchronous.  There is no CPU fallback: every call either runs on the
 * GPU or returns a negative status.
 *
 * level is 2, 3 or 5 (params.hpp:53-55; runtime dispatch as with_params, params.hpp:91-106).
 * Byte sizes per level: pk 1312/1952/2592, sk 2528/4000/4864, sig 2420/3293/4595.
 *
 * level 44, 65 or 87 selects ML-DSA-44/65/87 (FIPS 204) on the same engine: the standard's
 * hashing conventions (H(xi||k||l), 64-byte tr, M' = 0||len||ctx||M with the context string of
 * dlb_set_mldsa_context, empty by default,
 * rho'' = H(K||0^32||mu) i.e. the deterministic variant, lambda/4-byte commitment hash).
 * Sizes: pk 1312/1952/2592, sk 2560/4032/4896, sig 2420/3309/4627.  Not part of the
 * reference (proj/README.md:120-121); pinned against OpenSSL, see oracle/dilithium_oracle.h.
 * rho_prime_override, where given, replaces rho'' (hedged signing: pass 64 fresh random bytes).
 *
 * Status codes: 0 ok; DLB_E_ARG bad argument; DLB_E_LEVEL unsupported level;
 * DLB_E_KEY malformed secret key (packing.hpp:79-86,215-233 -- the C++ shim turns this
 * into std::invalid_argument / nullopt); <= -1000: -(1000 + cudaError_t).
 */
#ifndef DILITHIUM_B200_H
#define DILITHIUM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DLB_OK 0
#define DLB_E_ARG (-1)
#define DLB_E_LEVEL (-2)
#define DLB_E_KEY (-3)
#define DLB_E_NOMEM (-4)
#define DLB_E_BUSY (-5)     /* the batch submitted 32 tickets ago is still un-waited: wait for it first */
#define DLB_E_INTERNAL (-6) /* a submitted batch was never completed (device fault) */

typedef struct dlb_ctx dlb_ctx;

/* BatchStats (batch.hpp:31-38) + device-scheduler counters. */
typedef struct dlb_sign_stats {
  uint64_t rounds;               /* scheduler rounds summed over all CTAs */
  uint64_t attempts;             /* executed attempts incl. speculative waste */
  uint64_t speculative;          /* attempts beyond a task's next unresolved nonce */
  uint64_t idle_slot_rounds;     /* slot-rounds that ran no attempt */
  uint64_t accepted_attempt_sum; /* sum over tasks of the winning attempt ordinal */
  uint64_t failed_tasks;         /* nonce space exhausted (scheduler.hpp:52,122-128) */
  /* device clock (%globaltimer, ns) of the scheduler kernel: first / last CTA start and exit */
  uint64_t t_first_start_ns, t_last_start_ns, t_first_exit_ns, t_last_exit_ns;
} dlb_sign_stats;

/* Library / device ------------------------------------------------------------------ */

/* Creates an engine on CUDA device `device`.  max_batch is a sizing hint: 0 = everything grows
 * on demand; > 0 = the signing state and the per-task arenas of that many tasks are built here
 * instead of inside the first call.  Replaces the per-call WorkerPool + MemoryPool construction of
 * batch.hpp:62-67 with a context that is built once and reused. */
int dlb_create(dlb_ctx** out, int device, size_t max_batch);
void dlb_destroy(dlb_ctx* ctx);
const char* dlb_version(void);
/* Device time (ms, CUDA events on the engine's stream) of the kernels of the last batch
 * call, excluding host<->device copies. */
float dlb_last_kernel_ms(const dlb_ctx* ctx);
/* Device time (ms) of the dominant kernel of the last sign call (k_sign_persistent). */
float dlb_last_main_kernel_ms(const dlb_ctx* ctx);
/* Number of kernel launches issued by the last batch call. */
unsigned dlb_last_launches(const dlb_ctx* ctx);
/* Use an external CUDA stream (e.g. the caller's current stream) for the *_dev entry
 * points; NULL restores the engine's own stream. */
int dlb_set_stream(dlb_ctx* ctx, void* cuda_stream);

/* INT32 issue-rate microbenchmark (roofline denominator for this path): out[0] LOP3,
 * out[1] IMAD, out[2] SHF, out[3] LOP3+IMAD interleaved, in 10^12 lane-operations/s. */
int dlb_measure_int32_peak(dlb_ctx* ctx, double out[4]);
/* out[0] mul.hi.s32 (IMAD.HI), out[1] mul.wide.s32 (IMAD.WIDE), same unit. */
int dlb_measure_imad_hi_peak(dlb_ctx* ctx, double out[2]);

/* Per-round scheduler trace (BatchConfig::trace, RoundTrace scheduler.hpp:21-28; the tool's
 * --trace CSV, dilithium_cli.cpp:128-134).  The device scheduler runs one independent round
 * loop per CTA, so a record is one round of one CTA: `stream` is the CTA, `round` its round
 * counter, the other fields as in RoundTrace restricted to that CTA's tasks and slots.
 * dlb_set_trace(ctx, cap): the next sign calls log up to cap records (0 switches the trace
 * off; default off -- logging costs one 32-byte store per CTA round).  dlb_get_trace copies
 * the records of the last sign call, in no particular order, and returns how many the call
 * produced (which may exceed cap: the surplus was dropped). */
typedef struct dlb_round_trace {
  uint32_t stream, round, unfinished, assigned, speculative, idle_slots, newly_done, reserved;
} dlb_round_trace;
int dlb_set_trace(dlb_ctx* ctx, size_t cap);
long long dlb_get_trace(dlb_ctx* ctx, dlb_round_trace* out, size_t max_records);

/* Per-attempt execution log (BatchConfig::assignment_hook, batch.hpp:28,87-88; Assignment
 * scheduler.hpp:14-19): one record per (task, attempt) the device scheduler actually ran,
 * speculative ones included.  `slot` is the global attempt slot (CTA * 128 + slot in the CTA),
 * `kappa` the first mask nonce of the attempt (attempt * l).  dlb_set_assignment_log(ctx, cap):
 * the next synchronous sign calls log up to cap records (0 = off, the default; logging costs
 * one atomic and one 16-byte store per executed attempt).  dlb_get_assignment_log copies the
 * records of the last sign call, in no particular order, and returns how many it produced. */
typedef struct dlb_assignment {
  uint32_t slot, task, attempt, kappa;
} dlb_assignment;
int dlb_set_assignment_log(dlb_ctx* ctx, size_t cap);
long long dlb_get_assignment_log(dlb_ctx* ctx, dlb_assignment* out, size_t max_records);

/* FIPS 204 context string for the ML-DSA levels (44 / 65 / 87): signing and verification
 * hash M' = 0 || len || ctx || M.  len <= 255; the default is the empty string.  Sticky per
 * context until changed; ignored by the round-3 levels.  DLB_E_BUSY while signing batches are in
 * flight (they hash their tasks with the current string). */
int dlb_set_mldsa_context(dlb_ctx* ctx, const uint8_t* context_string, size_t len);
/* HashML-DSA (FIPS 204 Alg. 4 / 5, the pre-hash variant): with a hash OID set (the DER encoding,
 * 11 bytes for the SHA-2 / SHA-3 / SHAKE identifiers of the standard, at most 16) signing and
 * verification hash M' = 1 || len || ctx || OID || m, where the "message" m each task passes is the
 * digest PH(M) the caller computed with that hash.  oid_len == 0 returns to pure ML-DSA
 * (dlb_set_mldsa_context).  Sticky per context; DLB_E_BUSY while signing batches are in flight. */
int dlb_set_mldsa_prehash(dlb_ctx* ctx, const uint8_t* context_string, size_t len, const uint8_t* oid,
                          size_t oid_len);

/* Several GPUs of one box: the transport limit is host memory and PCIe, so the host thread that
 * drives a GPU -- and the pinned staging it allocates -- should live on that GPU's NUMA node.
 * dlb_bind_thread_to_device pins the CALLING thread to the CPUs local to CUDA device `device`
 * (/sys/bus/pci/devices/<id>/local_cpulist); memory it allocates afterwards (dlb_host_alloc,
 * dlb_create's staging) is then node-local by first touch.  Returns 0 when the affinity was
 * set, 1 when the box exposes no locality information (nothing changed), < 0 on errors.
 * dlb_device_numa_node: the node id, or -1 when unknown. */
int dlb_bind_thread_to_device(int device);
int dlb_device_numa_node(int device);

/* Pinned host memory for callers that want zero-staging transfers (the engine copies
 * straight from/to these buffers with cudaMemcpyAsync). */
void* dlb_host_alloc(size_t bytes);
void dlb_host_free(void* p);

/* Host-buffer batch API (what batch.hpp binds) ----------------------------------------- */

/* batch_keygen<P>(zetas, workers)  batch.hpp:159-166 / keygen<P>  scheme.hpp:68-104.
 * zetas: n*32 bytes.  pks: n*pk_bytes.  sks: n*sk_bytes. */
int dlb_keygen_batch(dlb_ctx* ctx, int level, size_t n, const uint8_t* zetas, uint8_t* pks,
                     uint8_t* sks);

/* batch_sign<P>(jobs, cfg, stats)  batch.hpp:53-137 (+ make_precomp scheme.hpp:106-125,
 * sign_with_precomp :253-266).
 *   sks, sk_stride: secret keys; sk_stride == 0 means one key shared by all tasks
 *                   (SignJob.key pointing at one SignPrecomp), else sks + i*sk_stride.
 *   msgs, msg_off:  messages concatenated; task i signs msgs[msg_off[i] .. msg_off[i+1]).
 *   rho_prime_override: NULL (deterministic signing) or n*64 bytes (scheme.hpp:253-258).
 *   psi:       resident attempt slots, BatchConfig::psi (0 = engine default).
 *   speculate: BatchConfig::speculate.  0 = one attempt per open task and round; 1 = idle
 *              slots run future nonces breadth first, at most 8 deep per round (measured
 *              optimum); N > 1 = the same with depth cap N.  Output never depends on it.
 *   sigs:      n*sig_bytes out.  attempts (nullable): winning attempt ordinal per task
 *              (SignOutput::attempts).  failed (nullable): 1 if the nonce space was
 *              exhausted (BatchStats::failed_tasks).  stats nullable.
 * Returns DLB_E_KEY if any secret key is malformed (no signature is produced). */
int dlb_sign_batch(dlb_ctx* ctx, int level, size_t n, const uint8_t* sks, size_t sk_stride,
                   const uint8_t* msgs, const uint64_t* msg_off,
                   const uint8_t* rho_prime_override, size_t psi, int speculate, uint8_t* sigs,
                   uint32_t* attempts, uint8_t* failed, dlb_sign_stats* stats);

/* batch_verify<P>(jobs, workers)  batch.hpp:148-156 / verify<P>  scheme.hpp:277-318.
 *   pks, pk_stride: pk_stride == 0 means one shared public key.
 *   sigs: n*sig_bytes (sig_stride = sig_bytes).  Tasks whose pk/sig length is wrong are
 *   the shim's business (flag 0 without touching the GPU, scheme.hpp:280-283); here
 *   every task has full-size inputs.
 *   flags: n bytes out, 1 accept / 0 reject.  Never fails per task otherwise. */
int dlb_verify_batch(dlb_ctx* ctx, int level, size_t n, const uint8_t* pks, size_t pk_stride,
                     const uint8_t* msgs, const uint64_t* msg_off, const uint8_t* sigs,
                     uint8_t* flags);

/* Mixed-key batches --------------------------------------------------------------------
 * batch.hpp:41-44: every SignJob carries a pointer to a caller-owned SignPrecomp and jobs
 * may share keys arbitrarily (a signing service multiplexing tenants).  The keyed forms
 * take the DISTINCT keys once (n_keys * sk_bytes / pk_bytes, contiguous) plus one 32-bit
 * key index per task, so make_precomp's work (ExpandA: 80/150/280 permutations, the NTTs
 * of s1, s2, t0; scheme.hpp:106-125) is done once per key on the device instead of once
 * per task.  key_idx[i] >= n_keys is DLB_E_ARG.  Everything else as the plain forms. */
int dlb_sign_batch_keyed(dlb_ctx* ctx, int level, size_t n_keys, const uint8_t* sks, size_t n,
                         const uint32_t* key_idx, const uint8_t* msgs, const uint64_t* msg_off,
                         const uint8_t* rho_prime_override, size_t psi, int speculate,
                         uint8_t* sigs, uint32_t* attempts, uint8_t* failed, dlb_sign_stats* stats);
int dlb_verify_batch_keyed(dlb_ctx* ctx, int level, size_t n_keys, const uint8_t* pks, size_t n,
                           const uint32_t* key_idx, const uint8_t* msgs, const uint64_t* msg_off,
                           const uint8_t* sigs, uint8_t* flags);

/* Batches in flight --------------------------------------------------------------------
 * The paper keeps several batches in flight per GPU (the reference
 * tool's engines, tools/dilithium_cli.cpp:309-345).  dlb_sign_submit enqueues a batch and
 * returns at once with a ticket; dlb_sign_wait blocks until that batch is complete and fills
 * the outputs.  Tickets are numbered consecutively (synchronous sign calls take one too) and the
 * engine keeps 32 consecutive tickets: a submission returns DLB_E_BUSY while the batch submitted 32
 * tickets earlier has not been waited for.  The device
 * scheduler is shared: CTAs that run out of tasks of one batch claim tasks of the next
 * submitted batches (of the same level) before they speculate, so the rejection-loop tail of a
 * batch overlaps the body of its successors.  Batches of different levels are served first come
 * first served.  Throughput grows with the work in flight until the scheduler's queues never run
 * dry: a batch's unluckiest task needs ~45 rounds, so a batch completes 55-100 ms after it was
 * submitted, and a steady stream wants about that much work in flight (100,000-task batches: 16;
 * measured 14.7 M sign/s against 14.3 at 8 and 10.6 one at a time).  Output bytes never depend
 * on what else is in flight.  Arguments as dlb_sign_batch / dlb_sign_batch_keyed (key_idx == NULL: sk_stride 0 =
 * one shared key, else one key per task; key_idx != NULL: a table of n_keys keys, sk_stride
 * = sk_bytes).  All input and output buffers must stay valid until the wait returns; a
 * signature buffer in pinned memory (dlb_host_alloc) is written in place by the device.
 * *ticket == 0 means the batch was empty (waiting on it returns at once).  Tickets may be
 * waited in any order.  The synchronous calls above are submit + wait. */
int dlb_sign_submit(dlb_ctx* ctx, int level, size_t n_keys, const uint8_t* sks, size_t sk_stride,
                    size_t n, const uint32_t* key_idx, const uint8_t* msgs, const uint64_t* msg_off,
                    const uint8_t* rho_prime_override, size_t psi, int speculate, uint8_t* sigs,
                    uint32_t* attempts, uint8_t* failed, uint64_t* ticket);
int dlb_sign_wait(dlb_ctx* ctx, uint64_t ticket, dlb_sign_stats* stats);
/* The same with every buffer in device memory. */
int dlb_sign_submit_dev(dlb_ctx* ctx, int level, size_t n_keys, const uint8_t* d_sks, size_t sk_stride,
                        size_t n, const uint32_t* d_key_idx, const uint8_t* d_msgs,
                        const uint64_t* d_msg_off, const uint8_t* d_rho_prime_override, size_t psi,
                        int speculate, uint8_t* d_sigs, uint32_t* d_attempts, uint8_t* d_failed,
                        uint64_t* ticket);

/* Device-resident variants -------------------------------------------------------------
 * Same contracts with every buffer already in device memory (HBM); no copies are made.
 * Used for kernel-only timing and by callers that keep keys/messages on the GPU. */
int dlb_keygen_batch_dev(dlb_ctx* ctx, int level, size_t n, const uint8_t* d_zetas,
                         uint8_t* d_pks, uint8_t* d_sks);
int dlb_sign_batch_dev(dlb_ctx* ctx, int level, size_t n, const uint8_t* d_sks, size_t sk_stride,
                       const uint8_t* d_msgs, const uint64_t* d_msg_off,
                       const uint8_t* d_rho_prime_override, size_t psi, int speculate,
                       uint8_t* d_sigs, uint32_t* d_attempts, uint8_t* d_failed,
                       dlb_sign_stats* stats /* host */);
int dlb_verify_batch_dev(dlb_ctx* ctx, int level, size_t n, const uint8_t* d_pks,
                         size_t pk_stride, const uint8_t* d_msgs, const uint64_t* d_msg_off,
                         const uint8_t* d_sigs, uint8_t* d_flags);

int dlb_sign_batch_keyed_dev(dlb_ctx* ctx, int level, size_t n_keys, const uint8_t* d_sks, size_t n,
                             const uint32_t* d_key_idx, const uint8_t* d_msgs,
                             const uint64_t* d_msg_off, const uint8_t* d_rho_prime_override,
                             size_t psi, int speculate, uint8_t* d_sigs, uint32_t* d_attempts,
                             uint8_t* d_failed, dlb_sign_stats* stats /* host */);
int dlb_verify_batch_keyed_dev(dlb_ctx* ctx, int level, size_t n_keys, const uint8_t* d_pks,
                               size_t n, const uint32_t* d_key_idx, const uint8_t* d_msgs,
                               const uint64_t* d_msg_off, const uint8_t* d_sigs, uint8_t* d_flags);

/* Stage-level entry points (device parity tests; host buffers) --------------------------
 * They run the same device functions the batch kernels use. */
int dlb_dbg_keccak_f1600(dlb_ctx* ctx, size_t n, uint64_t* states /* n*25, in place */);
int dlb_dbg_shake256(dlb_ctx* ctx, size_t n, const uint8_t* msgs, const uint64_t* msg_off,
                     uint8_t* out64 /* n*64: first 64 output bytes */);
int dlb_dbg_expand_a(dlb_ctx* ctx, int level, size_t n_keys, const uint8_t* rhos /* n*32 */,
                     int32_t* out /* n*K*L*256 */);
int dlb_dbg_expand_s(dlb_ctx* ctx, int level, size_t n, const uint8_t* rho_primes /* n*64 */,
                     int8_t* out /* n*(L+K)*256 */);
int dlb_dbg_expand_mask(dlb_ctx* ctx, int level, size_t n, const uint8_t* rho_primes /* n*64 */,
                        const uint32_t* kappas /* n */, int32_t* out /* n*L*256 */);
int dlb_dbg_sample_in_ball(dlb_ctx* ctx, int level, size_t n, const uint8_t* c_tildes /* n*32 */,
                           int8_t* out /* n*256 */);
/* rounding.hpp:13-59 for the n values first, first+1, ... (canonical, in [0,q)) with
 * gamma2 = (q-1)/gamma2_divisor (88 or 32).  out6: six arrays of n: Power2Round high, low;
 * Decompose high, low; UseHint with hint 0, hint 1. */
int dlb_dbg_rounding(dlb_ctx* ctx, int gamma2_divisor, int32_t first, size_t n, int32_t* out6);
/* forward NTT (output canonical [0,q)) and inverse NTT of canonical input (output
 * canonical): value-level parity with ntt.hpp:74-126.  inverse = 2: the input is used as
 * given, any signed representatives in (-q, q) -- the range the kernels feed the inverse
 * transform with; exercises the lazy-reduction bound on its worst case. */
int dlb_dbg_ntt(dlb_ctx* ctx, size_t n, int32_t* polys /* n*256 in place */, int inverse);
/* sign_attempt<P> (scheme.hpp:225-230): one rejection-loop iteration per task at kappa[i].
 * accepted[i] 0/1; c_tilde n*32; z n*L*256 centered; hints n*K*256 -- the latter two
 * are meaningful for accepted attempts. */
int dlb_dbg_sign_attempt(dlb_ctx* ctx, int level, size_t n, const uint8_t* sks, size_t sk_stride,
                         const uint8_t* mus /* n*64 */, const uint8_t* rho_primes /* n*64 */,
                         const uint32_t* kappas, uint8_t* accepted, uint8_t* c_tilde, int32_t* z,
                         int32_t* hints);

/* detail::sign_attempt_bounded<P> (scheme.hpp:133-219): the same with the three norm bounds
 * injected (tests force individual reject stages through them; each must be in [0, (q-1)/8],
 * rounding.hpp:65).  stage[i]: 255 accepted, else the RejectStage (scheme.hpp:34) the reference
 * reports -- the first failing check in its order: 0 ZNorm, 1 R0Norm, 2 VtNorm, 3 HintWeight. */
int dlb_dbg_sign_attempt_bounded(dlb_ctx* ctx, int level, size_t n, const uint8_t* sks,
                                 size_t sk_stride, const uint8_t* mus, const uint8_t* rho_primes,
                                 const uint32_t* kappas, int32_t z_bound, int32_t r0_bound,
                                 int32_t vt_bound, uint8_t* accepted, uint8_t* stage, uint8_t* c_tilde,
                                 int32_t* z, int32_t* hints);
/* Shrinks the nonce space of the following sign calls: a task whose attempts 0 .. max_attempt
 * all fail is reported failed (scheduler.hpp:52,122-128 -- the real limit, (65535 - (l-1)) / l,
 * is never reached by honest inputs).  0 restores the scheme's limit. */
int dlb_dbg_set_max_attempt(dlb_ctx* ctx, unsigned max_attempt);

#ifdef __cplusplus
}
#endif
#endif
