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

// Rotations on the fma pipe.  A 64-bit rotate is two funnel shifts on the alu pipe, the pipe every
// other instruction of the permutation (LOP3) needs as well; the fma pipe idles.  hi:lo rotated
// left by r < 32 is {hi * 2^r + (lo >> (32 - r)), lo * 2^r + (hi >> (32 - r))}: two IMAD.WIDE by
// 2^r give all four terms ({x >> (32 - r), x << r} = x * 2^r as 64 bits), two more IMADs (or one
// IMAD and one LOP3) put them together.  The multipliers come from the constant bank, which keeps
// ptxas from turning the multiplies back into shifts.  DLB_KECCAK_FMA_ROT = how many of the 29
// rotations of a round go that way (0: none).
#ifndef DLB_KECCAK_FMA_ROT
#define DLB_KECCAK_FMA_ROT 0
#endif
__device__ __constant__ uint32_t kRotMul[33] = {
    1u << 0,  1u << 1,  1u << 2,  1u << 3,  1u << 4,  1u << 5,  1u << 6,  1u << 7,  1u << 8,  1u << 9,  1u << 10,
    1u << 11, 1u << 12, 1u << 13, 1u << 14, 1u << 15, 1u << 16, 1u << 17, 1u << 18, 1u << 19, 1u << 20, 1u << 21,
    1u << 22, 1u << 23, 1u << 24, 1u << 25, 1u << 26, 1u << 27, 1u << 28, 1u << 29, 1u << 30, 1u << 31, 1u};

template <int R>
__device__ __forceinline__ uint64_t rotl64_fma(uint64_t x) {
  static_assert(R % 32 != 0, "plain moves otherwise");
  uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
  if (R > 32) {
    const uint32_t t = lo;
    lo = hi;
    hi = t;
  }
  const uint32_t p = kRotMul[R & 31], one = kRotMul[32];
  uint32_t alo, ahi, blo, bhi, nlo, nhi;
  asm("{\n\t.reg .u64 w;\n\tmul.wide.u32 w, %2, %3;\n\tmov.b64 {%0, %1}, w;\n\t}" : "=r"(alo), "=r"(ahi) : "r"(lo), "r"(p));
  asm("{\n\t.reg .u64 w;\n\tmul.wide.u32 w, %2, %3;\n\tmov.b64 {%0, %1}, w;\n\t}" : "=r"(blo), "=r"(bhi) : "r"(hi), "r"(p));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(nlo) : "r"(alo), "r"(one), "r"(bhi));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(nhi) : "r"(blo), "r"(one), "r"(ahi));
  return ((uint64_t)nhi << 32) | nlo;
}

// rotation number IDX (0..28) of a round: on the fma pipe if IDX < DLB_KECCAK_FMA_ROT
template <int R, int IDX>
__device__ __forceinline__ uint64_t rotl64_sel(uint64_t x);

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

template <int R, int IDX>
__device__ __forceinline__ uint64_t rotl64_sel(uint64_t x) {
  if constexpr (R % 32 != 0 && IDX < DLB_KECCAK_FMA_ROT) return rotl64_fma<R>(x);
  else return rotl64<R>(x);
}

__device__ __forceinline__ void keccak_round(uint64_t (&s)[25], uint64_t rc) {
  uint64_t c[5], r[5], b[25];
#pragma unroll
  for (int x = 0; x < 5; ++x) c[x] = s[x] ^ s[x + 5] ^ s[x + 10] ^ s[x + 15] ^ s[x + 20];
  {
  r[0] = rotl64_sel<1, 24>(c[0]);
  r[1] = rotl64_sel<1, 25>(c[1]);
  r[2] = rotl64_sel<1, 26>(c[2]);
  r[3] = rotl64_sel<1, 27>(c[3]);
  r[4] = rotl64_sel<1, 28>(c[4]);
  }
  // theta + rho + pi: b[y + 5*((2x+3y)%5)] = rotl(s[x+5y] ^ d[x], rho[x+5y]) with
  // d[x] = c[x-1] ^ rotl(c[x+1], 1) folded into the same three-input XOR (one LOP3 per
  // 32-bit half instead of forming d first: 10 instructions fewer per round)
#define DLB_TH(i, x) (s[i] ^ c[((x) + 4) % 5] ^ r[((x) + 1) % 5])
  b[0] = rotl64<0>(DLB_TH(0, 0));
  b[10] = rotl64_sel<1, 0>(DLB_TH(1, 1));
  b[20] = rotl64_sel<62, 1>(DLB_TH(2, 2));
  b[5] = rotl64_sel<28, 2>(DLB_TH(3, 3));
  b[15] = rotl64_sel<27, 3>(DLB_TH(4, 4));
  b[16] = rotl64_sel<36, 4>(DLB_TH(5, 0));
  b[1] = rotl64_sel<44, 5>(DLB_TH(6, 1));
  b[11] = rotl64_sel<6, 6>(DLB_TH(7, 2));
  b[21] = rotl64_sel<55, 7>(DLB_TH(8, 3));
  b[6] = rotl64_sel<20, 8>(DLB_TH(9, 4));
  b[7] = rotl64_sel<3, 9>(DLB_TH(10, 0));
  b[17] = rotl64_sel<10, 10>(DLB_TH(11, 1));
  b[2] = rotl64_sel<43, 11>(DLB_TH(12, 2));
  b[12] = rotl64_sel<25, 12>(DLB_TH(13, 3));
  b[22] = rotl64_sel<39, 13>(DLB_TH(14, 4));
  b[23] = rotl64_sel<41, 14>(DLB_TH(15, 0));
  b[8] = rotl64_sel<45, 15>(DLB_TH(16, 1));
  b[18] = rotl64_sel<15, 16>(DLB_TH(17, 2));
  b[3] = rotl64_sel<21, 17>(DLB_TH(18, 3));
  b[13] = rotl64_sel<8, 18>(DLB_TH(19, 4));
  b[14] = rotl64_sel<18, 19>(DLB_TH(20, 0));
  b[24] = rotl64_sel<2, 20>(DLB_TH(21, 1));
  b[9] = rotl64_sel<61, 21>(DLB_TH(22, 2));
  b[19] = rotl64_sel<56, 22>(DLB_TH(23, 3));
  b[4] = rotl64_sel<14, 23>(DLB_TH(24, 4));
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
