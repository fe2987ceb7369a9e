// chacha.cuh -- ChaCha ARX core for sm_100a.
//
// The quarter round is the reference's (pkg/src/pagecrypt/_chacha_numba.py:27-41):
//   a+=b; d^=a; d<<<=16;  c+=d; b^=c; b<<<=12;  a+=b; d^=a; d<<<=8;  c+=d; b^=c; b<<<=7
// with native 32-bit arithmetic instead of the reference's uint64-and-mask
// emulation (_chacha_numba.py:11,29-40).  Rotates by 16 and 8 are byte
// permutes (PRMT), 12 and 7 are funnel shifts (SHF.L.W): one ALU-pipe
// instruction each.
//
// Pipe balance.  IADD3/LOP3/SHF/PRMT all issue to the ALU pipe (16 lanes/clk
// per SMSP), IMAD to the FMA pipe.  A ChaCha quarter round is 4 adds + 4 xors
// + 4 rotates = 12 ALU ops if every add is an IADD3.  AddMode moves the adds to
// the FMA pipe as `mad.lo.u32 r, b, one, a` with `one` a runtime kernel
// argument equal to 1 (ptxas cannot fold it back into an IADD3), leaving
// 8 ALU + 4 FMA ops per quarter round.
#pragma once
#include <cstdint>

namespace pc {

enum AddMode : int {
  kAddAlu = 0,   // every add is IADD3 (ALU pipe)
  kAddFma = 1,   // every add is IMAD (FMA pipe)
  kAddSplitA = 2 // the two a+=b adds on the FMA pipe, c+=d on the ALU pipe
};

__device__ __forceinline__ uint32_t rotl16(uint32_t x) { return __byte_perm(x, 0, 0x1032); }
__device__ __forceinline__ uint32_t rotl8(uint32_t x) { return __byte_perm(x, 0, 0x2103); }
__device__ __forceinline__ uint32_t rotl12(uint32_t x) { return __funnelshift_l(x, x, 12); }
__device__ __forceinline__ uint32_t rotl7(uint32_t x) { return __funnelshift_l(x, x, 7); }

__device__ __forceinline__ uint32_t add_fma(uint32_t a, uint32_t b, uint32_t one) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(b), "r"(one), "r"(a));
  return r;
}

template <bool Fma>
__device__ __forceinline__ uint32_t add(uint32_t a, uint32_t b, uint32_t one) {
  if constexpr (Fma) return add_fma(a, b, one);
  else return a + b;
}

template <int AM>
__device__ __forceinline__ void quarter_round(uint32_t &a, uint32_t &b, uint32_t &c, uint32_t &d,
                                              uint32_t one) {
  constexpr bool fa = (AM == kAddFma) || (AM == kAddSplitA);
  constexpr bool fc = (AM == kAddFma);
  a = add<fa>(a, b, one); d = rotl16(d ^ a);
  c = add<fc>(c, d, one); b = rotl12(b ^ c);
  a = add<fa>(a, b, one); d = rotl8(d ^ a);
  c = add<fc>(c, d, one); b = rotl7(b ^ c);
}

// ROUNDS single rounds = ROUNDS/2 double rounds (column then diagonal),
// _chacha_numba.py:68-76.
template <int ROUNDS, int AM>
__device__ __forceinline__ void chacha_rounds(uint32_t (&x)[16], uint32_t one) {
  static_assert(ROUNDS % 2 == 0, "rounds must be even");
#pragma unroll
  for (int i = 0; i < ROUNDS / 2; ++i) {
    quarter_round<AM>(x[0], x[4], x[8], x[12], one);
    quarter_round<AM>(x[1], x[5], x[9], x[13], one);
    quarter_round<AM>(x[2], x[6], x[10], x[14], one);
    quarter_round<AM>(x[3], x[7], x[11], x[15], one);
    quarter_round<AM>(x[0], x[5], x[10], x[15], one);
    quarter_round<AM>(x[1], x[6], x[11], x[12], one);
    quarter_round<AM>(x[2], x[7], x[8], x[13], one);
    quarter_round<AM>(x[3], x[4], x[9], x[14], one);
  }
}

constexpr uint32_t kSigma0 = 0x61707865u; // "expa"
constexpr uint32_t kSigma1 = 0x3320646eu; // "nd 3"
constexpr uint32_t kSigma2 = 0x79622d32u; // "2-by"
constexpr uint32_t kSigma3 = 0x6b206574u; // "te k"

// Full block function: x := ChaCha_R(init) + init  (feed-forward,
// _chacha_numba.py:77-93).  k[8] key words, s[4] = state words 12..15.
template <int ROUNDS, int AM>
__device__ __forceinline__ void chacha_block(uint32_t (&x)[16], const uint32_t (&k)[8],
                                             const uint32_t (&s)[4], uint32_t one) {
  x[0] = kSigma0; x[1] = kSigma1; x[2] = kSigma2; x[3] = kSigma3;
#pragma unroll
  for (int i = 0; i < 8; ++i) x[4 + i] = k[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) x[12 + i] = s[i];
  chacha_rounds<ROUNDS, AM>(x, one);
  x[0] += kSigma0; x[1] += kSigma1; x[2] += kSigma2; x[3] += kSigma3;
#pragma unroll
  for (int i = 0; i < 8; ++i) x[4 + i] += k[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) x[12 + i] += s[i];
}

} // namespace pc
