// sign_queue.cuh -- device-visible state of the signing scheduler that the host context owns:
// the ring of in-flight batch descriptors and the log counters.  (Reference roles:
// scheduler.hpp:44-186 task LUT / batch.hpp:53-137 batch bookkeeping; PAPER.md:710-721 batches in flight.)
#pragma once
#include <cstdint>

namespace dlb {

constexpr int kRing = 32;    // batch descriptors per context = consecutive tickets that may be in flight
constexpr int kLanes = 4;    // stream lanes / scratch sets; a ticket's kernel takes the lowest idle lane, else T % kLanes

struct SignBatch {
  // ---- immutable once published (copied into shared memory by every CTA that serves it)
  unsigned n;                 // tasks
  unsigned tcap;              // max tasks of this batch a CTA holds at a time
  unsigned max_attempt;       // (65535 - (L-1)) / L   (scheduler.hpp:52)
  unsigned spec_depth;        // deepest speculative attempt per task and round; 0 = no speculation
  unsigned key_stride;        // 0 shared key, 1 per-task keys (when key_idx == nullptr)
  int level;                  // parameter set the batch was submitted for
  unsigned exclusive;         // stage-test batches: served by their own kernel only
  unsigned ticket1;           // ticket + 1
  const uint64_t* mu;         // n * 8
  const uint64_t* rho_prime;  // n * 8
  const uint32_t* kappa0;     // nullable: first nonce per task (stage tests)
  const int32_t* A;           // keys * K*L*256
  const int32_t* shat;        // keys * (L+2K)*256
  const uint32_t* key_idx;    // nullable: key table index of each task
  uint8_t* sigs;              // n * sig_bytes (device memory or mapped pinned host memory)
  uint32_t* attempts_out;     // nullable
  uint8_t* failed_out;        // nullable
  uint8_t* dbg_ctilde;        // nullable: n * CT, c~ of each task's first executed attempt
  uint8_t* dbg_stage;         // nullable: n, reject stage of the single-round attempt (DBG kernel)
  // message digests are computed by the scheduler itself when a CTA claims a task (no kernel of
  // the next batch has to find room beside a fully resident scheduler grid): msg_off != nullptr
  const uint8_t* sk_base;     // packed secret keys (tr at +64, K at +32), sk_bytes apart
  const uint8_t* msgs;        // concatenated messages
  const uint64_t* msg_off;    // n + 1 offsets; nullptr = mu / rho' supplied (stage tests)
  const uint8_t* pfx;         // FIPS 204: 0 || |ctx| || ctx
  unsigned plen;
  unsigned pad3;
  uint64_t* mu_w;             // where the digests go (= mu, rho_prime; rp_w null with an override)
  uint64_t* rp_w;
  int32_t bounds[3];          // DBG kernel: z, r0, c*t0 norm bounds (scheme.hpp:133-138)
  unsigned pad0;
  volatile unsigned* host_flag;  // mapped pinned word: set to ticket + 1 when done == n
  // per-key precomputation done by the scheduler itself (keys that are not in the cross-call cache:
  // key tables, one key per task): prep_n keys at prep_sks + k * prep_stride -> A, shat above.  The
  // batch's tasks become claimable when prep_done == prep_n.
  const uint8_t* prep_sks;
  unsigned prep_stride;
  unsigned prep_n;
  unsigned stage_out;         // signatures always go through the staging buffer and one whole-row copy (DLB_HOST_STAGE)
  unsigned pad4;
  // ---- mutable (device atomics)
  unsigned long long head;    // the device work queue of this batch: (ticket + 1) << 32 | next unclaimed
                              // task; claimed by compare-and-swap, so a stale view can never claim
  unsigned long long prep_q;  // (ticket + 1) << 32 | next key to precompute, claimed like `head`
  unsigned prep_done;         // keys precomputed
  unsigned pad1;
  unsigned done;              // committed tasks
  unsigned key_bad;           // some secret key failed the eta range check
  unsigned long long rounds, attempts, speculative, idle_slots, accepted_sum, failed;
  // %globaltimer, ns: first / last claim of a task, first / last commit of a task
  unsigned long long t_first_start, t_last_start, t_first_exit, t_last_exit;
  // ---- gate: written by a second, later copy; ticket + 1 = descriptor complete
  unsigned gate;
  unsigned pad2;
};

struct SignLog {  // per-context device counters of the optional logs
  unsigned long long trace_count;  // per-round trace records produced (may exceed the capacity)
  unsigned long long alog_count;   // executed-attempt records produced (may exceed the capacity)
};

}  // namespace dlb
