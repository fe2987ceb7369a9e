// chacha.cuh -- ChaCha ARX core for sm_100a.
//
// The quarter round is the reference's (pkg/src/pagecrypt/_chacha_numba.py:27-41):
//   a+=b; d^=a; d<<<=16;  c+=d; b^=c; b<<<=12;  a+=b; d^=a; d<<<=8;  c+=d; b^=c; b<<<=7
// with native 32-bit arithmetic instead of the reference's uint64-and-mask
// emulation (_chacha_numba.py:11,29-40).  Rotates by 16 and 8 are byte
// permutes (PRMT), 12 and 7 are funnel shifts (SHF.L.W): one ALU-pipe
// instruction each.
//
// Pipe balance.  IADD3/LOP3/SHF/PRMT issue to the ALU pipe (16 lanes/clk per
// SMSP), IMAD to the FMA pipe.  ptxas already emits the quarter round's adds
// as IMAD.IADD, leaving 4 xors + 4 rotates = 8 ALU ops against 4 FMA ops per
// quarter round: the ALU pipe is the binding constraint.  ROTMASK moves
// selected rotates to the FMA pipe as  lo = x * 2^n ; r = mulhi(x, 2^n) + lo
// (IMAD + IMAD.HI, with 2^n a runtime kernel argument so ptxas cannot turn
// the multiply back into a shift).  ROTMASK holds one nibble per quarter
// round of a double round (QR0 = lowest nibble: the four column rounds, then
// the four diagonal rounds); nibble bit 0/1/2/3 offloads the rotate by
// 16/12/8/7.
#pragma once
#include <cstdint>

namespace pc {

// Runtime multipliers 2^16, 2^12, 2^8, 2^7 for FMA-pipe rotates.
struct RotMul {
  uint32_t m16, m12, m8, m7;
};

__device__ __forceinline__ uint32_t rotl16(uint32_t x) { return __byte_perm(x, 0, 0x1032); }
__device__ __forceinline__ uint32_t rotl8(uint32_t x) { return __byte_perm(x, 0, 0x2103); }
__device__ __forceinline__ uint32_t rotl12(uint32_t x) { return __funnelshift_l(x, x, 12); }
__device__ __forceinline__ uint32_t rotl7(uint32_t x) { return __funnelshift_l(x, x, 7); }

// rotl(x, n) on the FMA pipe: (x << n) + (x >> (32 - n)) = lo(x*2^n) + hi(x*2^n)
// = IMAD(x, 2^n, IMAD.HI(x, 2^n, 0)): two FMA-pipe instructions.
__device__ __forceinline__ uint32_t rotl_fma(uint32_t x, uint32_t pow2) {
  uint32_t hi, r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(hi) : "r"(x), "r"(pow2));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(pow2), "r"(hi));
  return r;
}

template <int N, bool Fma>
__device__ __forceinline__ uint32_t rot(uint32_t x, uint32_t pow2) {
  if constexpr (Fma) return rotl_fma(x, pow2);
  else if constexpr (N == 16) return rotl16(x);
  else if constexpr (N == 12) return rotl12(x);
  else if constexpr (N == 8) return rotl8(x);
  else return rotl7(x);
}

template <uint32_t NIB>
__device__ __forceinline__ void quarter_round(uint32_t &a, uint32_t &b, uint32_t &c, uint32_t &d,
                                              const RotMul &m) {
  a += b; d = rot<16, (NIB & 1) != 0>(d ^ a, m.m16);
  c += d; b = rot<12, (NIB & 2) != 0>(b ^ c, m.m12);
  a += b; d = rot<8, (NIB & 4) != 0>(d ^ a, m.m8);
  c += d; b = rot<7, (NIB & 8) != 0>(b ^ c, m.m7);
}

template <uint32_t MASK>
__device__ __forceinline__ void column_round(uint32_t (&x)[16], const RotMul &m) {
  quarter_round<(MASK >> 0) & 15>(x[0], x[4], x[8], x[12], m);
  quarter_round<(MASK >> 4) & 15>(x[1], x[5], x[9], x[13], m);
  quarter_round<(MASK >> 8) & 15>(x[2], x[6], x[10], x[14], m);
  quarter_round<(MASK >> 12) & 15>(x[3], x[7], x[11], x[15], m);
}

template <uint32_t MASK>
__device__ __forceinline__ void diagonal_round(uint32_t (&x)[16], const RotMul &m) {
  quarter_round<(MASK >> 16) & 15>(x[0], x[5], x[10], x[15], m);
  quarter_round<(MASK >> 20) & 15>(x[1], x[6], x[11], x[12], m);
  quarter_round<(MASK >> 24) & 15>(x[2], x[7], x[8], x[13], m);
  quarter_round<(MASK >> 28) & 15>(x[3], x[4], x[9], x[14], m);
}

// ROUNDS single rounds = ROUNDS/2 double rounds (column then diagonal),
// _chacha_numba.py:68-76.
template <int ROUNDS, uint32_t MASK>
__device__ __forceinline__ void chacha_rounds(uint32_t (&x)[16], const RotMul &m) {
  static_assert(ROUNDS % 2 == 0, "rounds must be even");
#pragma unroll
  for (int i = 0; i < ROUNDS / 2; ++i) {
    column_round<MASK>(x, m);
    diagonal_round<MASK>(x, m);
  }
}

constexpr uint32_t kSigma0 = 0x61707865u; // "expa"
constexpr uint32_t kSigma1 = 0x3320646eu; // "nd 3"
constexpr uint32_t kSigma2 = 0x79622d32u; // "2-by"
constexpr uint32_t kSigma3 = 0x6b206574u; // "te k"

// Full block function: x := ChaCha_R(init) + init  (feed-forward,
// _chacha_numba.py:77-93).  k[8] key words, s[4] = state words 12..15.
template <int ROUNDS, uint32_t MASK>
__device__ __forceinline__ void chacha_block(uint32_t (&x)[16], const uint32_t (&k)[8],
                                             const uint32_t (&s)[4], const RotMul &m) {
  x[0] = kSigma0; x[1] = kSigma1; x[2] = kSigma2; x[3] = kSigma3;
#pragma unroll
  for (int i = 0; i < 8; ++i) x[4 + i] = k[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) x[12 + i] = s[i];
  chacha_rounds<ROUNDS, MASK>(x, m);
  x[0] += kSigma0; x[1] += kSigma1; x[2] += kSigma2; x[3] += kSigma3;
#pragma unroll
  for (int i = 0; i < 8; ++i) x[4 + i] += k[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) x[12 + i] += s[i];
}

} // namespace pc
