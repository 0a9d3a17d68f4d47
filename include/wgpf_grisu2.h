/* wgpf_grisu2.h -- JSON number text exactly as the reference's JSON library
 * prints it (nlohmann/json 3.11.3, a dependency of the reference's
 * export_chrome_trace, trace.hpp:493-511; not vendored in /root/reference).
 *
 * Restated from the published algorithm: Grisu2 (F. Loitsch, "Printing
 * Floating-Point Numbers Quickly and Accurately with Integers", PLDI 2010)
 * with the boundary handling, cached-power selection (alpha = -60,
 * gamma = -32, powers 10^k for k = -300 .. 324 step 8) and round-weeding
 * step of that library's dtoa, then its layout rules: ".0" after integral
 * values, plain notation for decimal exponents in (-4, 15], otherwise
 * d.ddde+XX with at least two exponent digits.  Grisu2 is not always the
 * shortest round-trip string (std::to_chars is), so byte parity needs this
 * exact algorithm.  Header-only, __host__ __device__: the host exporter and
 * the GPU exporter (k_chrome.cuh) share it.  Table: scripts/gen_cached_powers.py.
 */
#ifndef WGPF_GRISU2_H
#define WGPF_GRISU2_H

#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define WGPF_HD __host__ __device__ __forceinline__
#else
#define WGPF_HD inline
#endif

namespace wgpf_json {

struct DiyFp {
  uint64_t f;
  int e;
};

struct CachedPower {
  uint64_t f;
  int e;
  int k;
};

WGPF_HD uint64_t mulhi_round(uint64_t x, uint64_t y) {
  /* high 64 bits of the 128-bit product, rounded half up at bit 63 */
#ifdef __CUDA_ARCH__
  const uint64_t hi = __umul64hi(x, y);
#else
  const uint64_t hi = (uint64_t)(((unsigned __int128)x * y) >> 64);
#endif
  return hi + ((x * y) >> 63);
}

WGPF_HD DiyFp mul(DiyFp a, DiyFp b) { return DiyFp{mulhi_round(a.f, b.f), a.e + b.e + 64}; }

WGPF_HD int clz64(uint64_t x) {
#ifdef __CUDA_ARCH__
  return __clzll((long long)x);
#else
  return __builtin_clzll(x);
#endif
}

WGPF_HD DiyFp normalize(DiyFp x) {
  const int s = clz64(x.f);
  return DiyFp{x.f << s, x.e - s};
}

/* 10^k ~= f * 2^e, k = -300 + 8 i, f normalised and rounded to nearest
 * (host and device copies of the same table) */
static const uint64_t kPow10F_host[79] = {
      0xAB70FE17C79AC6CAull,
      0xFF77B1FCBEBCDC4Full,
      0xBE5691EF416BD60Cull,
      0x8DD01FAD907FFC3Cull,
      0xD3515C2831559A83ull,
      0x9D71AC8FADA6C9B5ull,
      0xEA9C227723EE8BCBull,
      0xAECC49914078536Dull,
      0x823C12795DB6CE57ull,
      0xC21094364DFB5637ull,
      0x9096EA6F3848984Full,
      0xD77485CB25823AC7ull,
      0xA086CFCD97BF97F4ull,
      0xEF340A98172AACE5ull,
      0xB23867FB2A35B28Eull,
      0x84C8D4DFD2C63F3Bull,
      0xC5DD44271AD3CDBAull,
      0x936B9FCEBB25C996ull,
      0xDBAC6C247D62A584ull,
      0xA3AB66580D5FDAF6ull,
      0xF3E2F893DEC3F126ull,
      0xB5B5ADA8AAFF80B8ull,
      0x87625F056C7C4A8Bull,
      0xC9BCFF6034C13053ull,
      0x964E858C91BA2655ull,
      0xDFF9772470297EBDull,
      0xA6DFBD9FB8E5B88Full,
      0xF8A95FCF88747D94ull,
      0xB94470938FA89BCFull,
      0x8A08F0F8BF0F156Bull,
      0xCDB02555653131B6ull,
      0x993FE2C6D07B7FACull,
      0xE45C10C42A2B3B06ull,
      0xAA242499697392D3ull,
      0xFD87B5F28300CA0Eull,
      0xBCE5086492111AEBull,
      0x8CBCCC096F5088CCull,
      0xD1B71758E219652Cull,
      0x9C40000000000000ull,
      0xE8D4A51000000000ull,
      0xAD78EBC5AC620000ull,
      0x813F3978F8940984ull,
      0xC097CE7BC90715B3ull,
      0x8F7E32CE7BEA5C70ull,
      0xD5D238A4ABE98068ull,
      0x9F4F2726179A2245ull,
      0xED63A231D4C4FB27ull,
      0xB0DE65388CC8ADA8ull,
      0x83C7088E1AAB65DBull,
      0xC45D1DF942711D9Aull,
      0x924D692CA61BE758ull,
      0xDA01EE641A708DEAull,
      0xA26DA3999AEF774Aull,
      0xF209787BB47D6B85ull,
      0xB454E4A179DD1877ull,
      0x865B86925B9BC5C2ull,
      0xC83553C5C8965D3Dull,
      0x952AB45CFA97A0B3ull,
      0xDE469FBD99A05FE3ull,
      0xA59BC234DB398C25ull,
      0xF6C69A72A3989F5Cull,
      0xB7DCBF5354E9BECEull,
      0x88FCF317F22241E2ull,
      0xCC20CE9BD35C78A5ull,
      0x98165AF37B2153DFull,
      0xE2A0B5DC971F303Aull,
      0xA8D9D1535CE3B396ull,
      0xFB9B7CD9A4A7443Cull,
      0xBB764C4CA7A44410ull,
      0x8BAB8EEFB6409C1Aull,
      0xD01FEF10A657842Cull,
      0x9B10A4E5E9913129ull,
      0xE7109BFBA19C0C9Dull,
      0xAC2820D9623BF429ull,
      0x80444B5E7AA7CF85ull,
      0xBF21E44003ACDD2Dull,
      0x8E679C2F5E44FF8Full,
      0xD433179D9C8CB841ull,
      0x9E19DB92B4E31BA9ull};
static const int16_t kPow10E_host[79] = {
      -1060, -1034, -1007, -980, -954, -927, -901, -874, -847, -821,
      -794, -768, -741, -715, -688, -661, -635, -608, -582, -555,
      -529, -502, -475, -449, -422, -396, -369, -343, -316, -289,
      -263, -236, -210, -183, -157, -130, -103, -77, -50, -24,
      3, 30, 56, 83, 109, 136, 162, 189, 216, 242,
      269, 295, 322, 348, 375, 402, 428, 455, 481, 508,
      534, 561, 588, 614, 641, 667, 694, 720, 747, 774,
      800, 827, 853, 880, 907, 933, 960, 986, 1013};
#ifdef __CUDACC__
static __constant__ uint64_t kPow10F_dev[79] = {
      0xAB70FE17C79AC6CAull,
      0xFF77B1FCBEBCDC4Full,
      0xBE5691EF416BD60Cull,
      0x8DD01FAD907FFC3Cull,
      0xD3515C2831559A83ull,
      0x9D71AC8FADA6C9B5ull,
      0xEA9C227723EE8BCBull,
      0xAECC49914078536Dull,
      0x823C12795DB6CE57ull,
      0xC21094364DFB5637ull,
      0x9096EA6F3848984Full,
      0xD77485CB25823AC7ull,
      0xA086CFCD97BF97F4ull,
      0xEF340A98172AACE5ull,
      0xB23867FB2A35B28Eull,
      0x84C8D4DFD2C63F3Bull,
      0xC5DD44271AD3CDBAull,
      0x936B9FCEBB25C996ull,
      0xDBAC6C247D62A584ull,
      0xA3AB66580D5FDAF6ull,
      0xF3E2F893DEC3F126ull,
      0xB5B5ADA8AAFF80B8ull,
      0x87625F056C7C4A8Bull,
      0xC9BCFF6034C13053ull,
      0x964E858C91BA2655ull,
      0xDFF9772470297EBDull,
      0xA6DFBD9FB8E5B88Full,
      0xF8A95FCF88747D94ull,
      0xB94470938FA89BCFull,
      0x8A08F0F8BF0F156Bull,
      0xCDB02555653131B6ull,
      0x993FE2C6D07B7FACull,
      0xE45C10C42A2B3B06ull,
      0xAA242499697392D3ull,
      0xFD87B5F28300CA0Eull,
      0xBCE5086492111AEBull,
      0x8CBCCC096F5088CCull,
      0xD1B71758E219652Cull,
      0x9C40000000000000ull,
      0xE8D4A51000000000ull,
      0xAD78EBC5AC620000ull,
      0x813F3978F8940984ull,
      0xC097CE7BC90715B3ull,
      0x8F7E32CE7BEA5C70ull,
      0xD5D238A4ABE98068ull,
      0x9F4F2726179A2245ull,
      0xED63A231D4C4FB27ull,
      0xB0DE65388CC8ADA8ull,
      0x83C7088E1AAB65DBull,
      0xC45D1DF942711D9Aull,
      0x924D692CA61BE758ull,
      0xDA01EE641A708DEAull,
      0xA26DA3999AEF774Aull,
      0xF209787BB47D6B85ull,
      0xB454E4A179DD1877ull,
      0x865B86925B9BC5C2ull,
      0xC83553C5C8965D3Dull,
      0x952AB45CFA97A0B3ull,
      0xDE469FBD99A05FE3ull,
      0xA59BC234DB398C25ull,
      0xF6C69A72A3989F5Cull,
      0xB7DCBF5354E9BECEull,
      0x88FCF317F22241E2ull,
      0xCC20CE9BD35C78A5ull,
      0x98165AF37B2153DFull,
      0xE2A0B5DC971F303Aull,
      0xA8D9D1535CE3B396ull,
      0xFB9B7CD9A4A7443Cull,
      0xBB764C4CA7A44410ull,
      0x8BAB8EEFB6409C1Aull,
      0xD01FEF10A657842Cull,
      0x9B10A4E5E9913129ull,
      0xE7109BFBA19C0C9Dull,
      0xAC2820D9623BF429ull,
      0x80444B5E7AA7CF85ull,
      0xBF21E44003ACDD2Dull,
      0x8E679C2F5E44FF8Full,
      0xD433179D9C8CB841ull,
      0x9E19DB92B4E31BA9ull};
static __constant__ int16_t kPow10E_dev[79] = {
      -1060, -1034, -1007, -980, -954, -927, -901, -874, -847, -821,
      -794, -768, -741, -715, -688, -661, -635, -608, -582, -555,
      -529, -502, -475, -449, -422, -396, -369, -343, -316, -289,
      -263, -236, -210, -183, -157, -130, -103, -77, -50, -24,
      3, 30, 56, 83, 109, 136, 162, 189, 216, 242,
      269, 295, 322, 348, 375, 402, 428, 455, 481, 508,
      534, 561, 588, 614, 641, 667, 694, 720, 747, 774,
      800, 827, 853, 880, 907, 933, 960, 986, 1013};
#endif

WGPF_HD CachedPower cached_power(int i) {
#ifdef __CUDA_ARCH__
  return CachedPower{kPow10F_dev[i], (int)kPow10E_dev[i], -300 + 8 * i};
#else
  return CachedPower{kPow10F_host[i], (int)kPow10E_host[i], -300 + 8 * i};
#endif
}

/* Grisu2 digits of a finite value > 0: buf gets the digits, the return the
 * count, *dexp the decimal exponent (value ~= digits * 10^dexp). */
WGPF_HD int grisu2(char* buf, int* dexp, double value) {
  uint64_t bits;
  memcpy(&bits, &value, 8);
  const uint64_t kHidden = 1ull << 52;
  const uint64_t F = bits & (kHidden - 1);
  const int E = (int)(bits >> 52);
  const DiyFp v = E == 0 ? DiyFp{F, 1 - 1075} : DiyFp{F + kHidden, E - 1075};
  const bool lower_closer = F == 0 && E > 1;
  const DiyFp m_plus = normalize(DiyFp{2 * v.f + 1, v.e - 1});
  const DiyFp m_minus0 = lower_closer ? DiyFp{4 * v.f - 1, v.e - 2} : DiyFp{2 * v.f - 1, v.e - 1};
  const DiyFp m_minus = DiyFp{m_minus0.f << (m_minus0.e - m_plus.e), m_plus.e};
  const DiyFp w0 = normalize(v);
  /* cached power bringing the exponent into [alpha, gamma] = [-60, -32] */
  const int fe = -60 - m_plus.e - 1;
  const int k = (fe * 78913) / (1 << 18) + (fe > 0 ? 1 : 0);
  const int index = (300 + k + 7) / 8;
  const CachedPower cp = cached_power(index);
  const DiyFp c = DiyFp{cp.f, cp.e};
  const DiyFp w = mul(w0, c);
  const DiyFp wm = mul(m_minus, c);
  const DiyFp wp = mul(m_plus, c);
  const DiyFp Mm = DiyFp{wm.f + 1, wm.e};
  const DiyFp Mp = DiyFp{wp.f - 1, wp.e};
  int dec = -cp.k;
  /* digit generation */
  uint64_t delta = Mp.f - Mm.f;
  uint64_t dist = Mp.f - w.f;
  const int sh = -Mp.e;
  const uint64_t one = 1ull << sh;
  uint32_t p1 = (uint32_t)(Mp.f >> sh);
  uint64_t p2 = Mp.f & (one - 1);
  uint32_t pow10;
  int n;
  if (p1 >= 1000000000u) { pow10 = 1000000000u; n = 10; }
  else if (p1 >= 100000000u) { pow10 = 100000000u; n = 9; }
  else if (p1 >= 10000000u) { pow10 = 10000000u; n = 8; }
  else if (p1 >= 1000000u) { pow10 = 1000000u; n = 7; }
  else if (p1 >= 100000u) { pow10 = 100000u; n = 6; }
  else if (p1 >= 10000u) { pow10 = 10000u; n = 5; }
  else if (p1 >= 1000u) { pow10 = 1000u; n = 4; }
  else if (p1 >= 100u) { pow10 = 100u; n = 3; }
  else if (p1 >= 10u) { pow10 = 10u; n = 2; }
  else { pow10 = 1u; n = 1; }
  int len = 0;
  uint64_t rest = 0, ten = 0;
  bool done = false;
  while (n > 0) {
    const uint32_t d = p1 / pow10;
    p1 = p1 % pow10;
    buf[len++] = (char)('0' + d);
    --n;
    rest = ((uint64_t)p1 << sh) + p2;
    if (rest <= delta) {
      dec += n;
      ten = (uint64_t)pow10 << sh;
      done = true;
      break;
    }
    pow10 /= 10;
  }
  if (!done) {
    int m = 0;
    for (;;) {
      p2 *= 10;
      buf[len++] = (char)('0' + (p2 >> sh));
      p2 &= one - 1;
      ++m;
      delta *= 10;
      dist *= 10;
      if (p2 <= delta) break;
    }
    dec -= m;
    rest = p2;
    ten = one;
  }
  /* round weeding: move the last digit towards w while it stays inside */
  while (rest < dist && delta - rest >= ten &&
         (rest + ten < dist || dist - rest > rest + ten - dist)) {
    buf[len - 1]--;
    rest += ten;
  }
  *dexp = dec;
  return len;
}

/* The JSON text of a finite double; returns the length (<= 32). */
WGPF_HD int format_double(char* out, double x) {
  uint64_t bits;
  memcpy(&bits, &x, 8);
  int o = 0;
  if (bits >> 63) {
    out[o++] = '-';
    bits &= ~(1ull << 63);
    memcpy(&x, &bits, 8);
  }
  if (bits == 0) {
    out[o++] = '0';
    out[o++] = '.';
    out[o++] = '0';
    return o;
  }
  char d[24];
  int dexp;
  const int k = grisu2(d, &dexp, x);
  const int n = k + dexp;  /* position of the decimal point */
  if (k <= n && n <= 15) {
    for (int i = 0; i < k; ++i) out[o++] = d[i];
    for (int i = k; i < n; ++i) out[o++] = '0';
    out[o++] = '.';
    out[o++] = '0';
  } else if (0 < n && n <= 15) {
    for (int i = 0; i < n; ++i) out[o++] = d[i];
    out[o++] = '.';
    for (int i = n; i < k; ++i) out[o++] = d[i];
  } else if (-4 < n && n <= 0) {
    out[o++] = '0';
    out[o++] = '.';
    for (int i = 0; i < -n; ++i) out[o++] = '0';
    for (int i = 0; i < k; ++i) out[o++] = d[i];
  } else {
    out[o++] = d[0];
    if (k > 1) {
      out[o++] = '.';
      for (int i = 1; i < k; ++i) out[o++] = d[i];
    }
    out[o++] = 'e';
    int e = n - 1;
    out[o++] = e < 0 ? '-' : '+';
    if (e < 0) e = -e;
    if (e < 10) {
      out[o++] = '0';
      out[o++] = (char)('0' + e);
    } else if (e < 100) {
      out[o++] = (char)('0' + e / 10);
      out[o++] = (char)('0' + e % 10);
    } else {
      out[o++] = (char)('0' + e / 100);
      out[o++] = (char)('0' + (e / 10) % 10);
      out[o++] = (char)('0' + e % 10);
    }
  }
  return o;
}

/* Decimal text of an unsigned integer; returns the length. */
WGPF_HD int format_u64(char* out, uint64_t v) {
  char t[20];
  int n = 0;
  do {
    t[n++] = (char)('0' + v % 10);
    v /= 10;
  } while (v);
  for (int i = 0; i < n; ++i) out[i] = t[n - 1 - i];
  return n;
}

}  // namespace wgpf_json

#endif /* WGPF_GRISU2_H */
