// keccak.cuh -- Keccak-f[1600] / SHAKE for sm_100a, one sponge per thread.
//
// Semantics: proj/include/dilithium/keccak.hpp:70-93 (permutation), :98-172 (sponge,
// pad 0x1F..0x80, rates 168/136).  Mapping: a warp advances 32 independent sponges in
// lockstep, each lane holding its 25 lanes x 64 bit in 50 registers.  The alternative
// the paper uses (25 threads of a warp share ONE state) needs ~22 SHFL + ~12 ALU
// warp-instructions per round per state, i.e. ~6x the issue slots of this layout
// (180 LOP3/SHF per round per state, no shuffles, no idle lanes); with >= 10^4
// independent streams per batch there is no need to split a state across lanes.
// The round loop is kept rolled (one round body, 24 trips) so the body (~3 KB of
// SASS) stays in the instruction cache next to the sampler code around it.
#pragma once
#include "common.cuh"

namespace dlb {

__device__ __constant__ const uint64_t kKeccakRC[24] = {
    0x0000000000000001ull, 0x0000000000008082ull, 0x800000000000808aull, 0x8000000080008000ull,
    0x000000000000808bull, 0x0000000080000001ull, 0x8000000080008081ull, 0x8000000000008009ull,
    0x000000000000008aull, 0x0000000000000088ull, 0x0000000080008009ull, 0x000000008000000aull,
    0x000000008000808bull, 0x800000000000008bull, 0x8000000000008089ull, 0x8000000000008003ull,
    0x8000000000008002ull, 0x8000000000000080ull, 0x000000000000800aull, 0x800000008000000aull,
    0x8000000080008081ull, 0x8000000000008080ull, 0x0000000080000001ull, 0x8000000080008008ull};

template <int R>
__device__ __forceinline__ uint64_t rotl64(uint64_t x) {
  if (R == 0) return x;
  const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
  uint32_t nlo, nhi;
  if (R == 32) {
    nlo = hi;
    nhi = lo;
  } else if (R < 32) {
    nlo = __funnelshift_l(hi, lo, R);
    nhi = __funnelshift_l(lo, hi, R);
  } else {
    nlo = __funnelshift_l(lo, hi, (R - 32) & 31);
    nhi = __funnelshift_l(hi, lo, (R - 32) & 31);
  }
  return ((uint64_t)nhi << 32) | nlo;
}

__device__ __forceinline__ void keccak_round(uint64_t (&s)[25], uint64_t rc) {
  uint64_t c[5], r[5], b[25];
#pragma unroll
  for (int x = 0; x < 5; ++x) c[x] = s[x] ^ s[x + 5] ^ s[x + 10] ^ s[x + 15] ^ s[x + 20];
#pragma unroll
  for (int x = 0; x < 5; ++x) r[x] = rotl64<1>(c[x]);
  // theta + rho + pi: b[y + 5*((2x+3y)%5)] = rotl(s[x+5y] ^ d[x], rho[x+5y]) with
  // d[x] = c[x-1] ^ rotl(c[x+1], 1) folded into the same three-input XOR (one LOP3 per
  // 32-bit half instead of forming d first: 10 instructions fewer per round)
#define DLB_TH(i, x) (s[i] ^ c[((x) + 4) % 5] ^ r[((x) + 1) % 5])
  b[0] = rotl64<0>(DLB_TH(0, 0));
  b[10] = rotl64<1>(DLB_TH(1, 1));
  b[20] = rotl64<62>(DLB_TH(2, 2));
  b[5] = rotl64<28>(DLB_TH(3, 3));
  b[15] = rotl64<27>(DLB_TH(4, 4));
  b[16] = rotl64<36>(DLB_TH(5, 0));
  b[1] = rotl64<44>(DLB_TH(6, 1));
  b[11] = rotl64<6>(DLB_TH(7, 2));
  b[21] = rotl64<55>(DLB_TH(8, 3));
  b[6] = rotl64<20>(DLB_TH(9, 4));
  b[7] = rotl64<3>(DLB_TH(10, 0));
  b[17] = rotl64<10>(DLB_TH(11, 1));
  b[2] = rotl64<43>(DLB_TH(12, 2));
  b[12] = rotl64<25>(DLB_TH(13, 3));
  b[22] = rotl64<39>(DLB_TH(14, 4));
  b[23] = rotl64<41>(DLB_TH(15, 0));
  b[8] = rotl64<45>(DLB_TH(16, 1));
  b[18] = rotl64<15>(DLB_TH(17, 2));
  b[3] = rotl64<21>(DLB_TH(18, 3));
  b[13] = rotl64<8>(DLB_TH(19, 4));
  b[14] = rotl64<18>(DLB_TH(20, 0));
  b[24] = rotl64<2>(DLB_TH(21, 1));
  b[9] = rotl64<61>(DLB_TH(22, 2));
  b[19] = rotl64<56>(DLB_TH(23, 3));
  b[4] = rotl64<14>(DLB_TH(24, 4));
#undef DLB_TH
  // chi
#pragma unroll
  for (int y = 0; y < 25; y += 5) {
#pragma unroll
    for (int x = 0; x < 5; ++x) s[y + x] = b[y + x] ^ (~b[y + (x + 1) % 5] & b[y + (x + 2) % 5]);
  }
  s[0] ^= rc;  // iota
}

__device__ __forceinline__ void keccak_f1600(uint64_t (&s)[25]) {
#pragma unroll 1
  for (int r = 0; r < 24; ++r) keccak_round(s, kKeccakRC[r]);
}

__device__ __forceinline__ void keccak_clear(uint64_t (&s)[25]) {
#pragma unroll
  for (int i = 0; i < 25; ++i) s[i] = 0;
}

constexpr int kRate128 = 168, kRate256 = 136;  // keccak.hpp:14-15
constexpr int kWords128 = 21, kWords256 = 17;

// 8 message bytes at offset `off` of a virtual message of total length `len` held at
// `p` (global, any alignment), zero beyond the end, with the SHAKE suffix 0x1F at
// byte `len` -- i.e. the word to XOR into the state for a padded message.  The final
// 0x80 is XORed by the caller into the last word of the block that holds byte `len`.
template <bool NC = true>
__device__ __forceinline__ uint64_t padded_word(const uint8_t* p, size_t len, size_t off) {
  uint64_t w = 0;
  if (off + 8 <= len) {
    w = (uint64_t)load_u32_unaligned<NC>(p + off) | ((uint64_t)load_u32_unaligned<NC>(p + off + 4) << 32);
  } else if (off <= len) {
    const int n = (int)(len - off);  // 0..7 valid bytes
    for (int i = 0; i < n; ++i) w |= (uint64_t)(NC ? __ldg(p + off + i) : ld_weak(p + off + i)) << (8 * i);
    w |= (uint64_t)0x1F << (8 * n);
  }
  return w;
}

// Absorb an arbitrary-length message: the first PRE_WORDS 64-bit words come from registers
// (`pre`), then `plen` bytes from `pfx` (global memory; FIPS 204's 0 || |ctx| || ctx in front
// of the message, plen = 0 for round 3), then msg[0..msg_len) from global memory.
// Leaves the sponge finalized and permuted once: s holds the first squeeze block.
template <int RATE_WORDS, int PRE_WORDS, bool NC = true>
__device__ __forceinline__ void shake_absorb_pre(uint64_t (&s)[25], const uint64_t (&pre)[PRE_WORDS],
                                                 const uint8_t* pfx, unsigned plen,
                                                 const uint8_t* msg, size_t msg_len) {
  static_assert(PRE_WORDS < RATE_WORDS, "prefix must fit the first block");
  keccak_clear(s);
  // the tail behind the register prefix is the virtual message  pfx || msg
  const size_t total = (size_t)PRE_WORDS * 8 + plen + msg_len;
  const size_t nblocks = total / (RATE_WORDS * 8) + 1;  // padding always adds a byte
  auto tail_word = [&](size_t off) -> uint64_t {  // 8 bytes of the padded tail at `off`
    if (plen == 0) return padded_word<NC>(msg, msg_len, off);
    if (off >= plen) return padded_word<NC>(msg, msg_len, off - plen);
    const unsigned nb = plen - (unsigned)off;  // prefix bytes from this word on
    if (nb >= 8)
      return (uint64_t)load_u32_unaligned<NC>(pfx + off) | ((uint64_t)load_u32_unaligned<NC>(pfx + off + 4) << 32);
    uint64_t w = 0;
    for (unsigned i = 0; i < nb; ++i) w |= (uint64_t)(NC ? __ldg(pfx + off + i) : ld_weak(pfx + off + i)) << (8 * i);
    return w | (padded_word<NC>(msg, msg_len, 0) << (8 * nb));  // the bytes shifted out lead the next word
  };
#pragma unroll 1
  for (size_t blk = 0; blk < nblocks; ++blk) {
    const size_t base = blk * RATE_WORDS * 8;
#pragma unroll
    for (int w = 0; w < RATE_WORDS; ++w) {
      uint64_t v;
      if (w < PRE_WORDS) {
        v = blk == 0 ? pre[w] : tail_word(base + 8 * w - PRE_WORDS * 8);
      } else {
        v = tail_word(base + 8 * w - PRE_WORDS * 8);
      }
      s[w] ^= v;
    }
    if (blk == nblocks - 1) s[RATE_WORDS - 1] ^= 0x8000000000000000ull;
    keccak_f1600(s);
  }
}

}  // namespace dlb
