// Band-image decode for load_stack / load_image (stack.py:119-177,
// rendering.py:334-343): the strips of a TIFF, staged to HBM as raw file bytes,
// become sample planes on the device.
//
// The reference decodes with cv2.imread (libtiff + zlib, one core).  A TIFF
// strip is an independent unit -- raw bytes, or its own zlib stream -- so the
// strips of a band are decoded in parallel:
//  * strips_copy_kernel: uncompressed strips, one CTA per strip (16-byte
//    vector copies when aligned);
//  * inflate_warp_kernel: deflate strips (Compression 8 / 32946) and PNG IDAT
//    streams, one warp per zlib stream: RFC 1951 stored / fixed / dynamic
//    blocks, 11-bit lookup tables with a canonical-walk fallback, a 32 KB
//    shared-memory history window, warp-wide match copies and flushes, Adler-32
//    verified (inflate_kernel, one thread per stream, is the first version,
//    kept behind UT_INFLATE_THREAD=1 for comparison);
//  * lzw_kernel: LZW strips / tiles (Compression 5, MSB-first codes of 9..12
//    bits with the TIFF "early change"), one thread per stream; a table entry is
//    (position, length) of the string's first occurrence in the stream's own
//    output, so the table costs 6 bytes per code and strings copy forward;
//  * unpredict_kernel: TIFF Predictor 2 (horizontal differencing) undone per
//    row and channel, after an optional byte swap of big-endian ('MM') 16-bit
//    samples;
//  * untile_kernel: decoded tiles (Tile* tags) scattered into the image rows;
//  * png_unfilter_kernel: the scanline filters of a PNG (None / Sub / Up /
//    Average / Paeth; the IDAT zlib stream is inflated by inflate_kernel), one
//    warp per image running a skewed wavefront over 32 rows at a time -- lane t
//    reconstructs row y0 + t one pixel behind lane t - 1, the "up" pixel arrives
//    by shuffle -- so the row-to-row and left-to-right dependencies of Average /
//    Paeth cost (width + 32) steps per 32 rows instead of 32 x width;
//    png_rows_kernel then drops the filter bytes and swaps 16-bit samples to
//    little endian.
// A stream whose data is malformed, too short or too long sets its status
// word (and the caller raises DataError, as cv2.imread failing does).
#include <cstdlib>

#include "common.cuh"

namespace ut {
namespace {

__constant__ uint16_t c_len_base[29] = {3,  4,  5,  6,  7,  8,  9,  10, 11,  13,  15,  17,  19,  23, 27,
                                        31, 35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
__constant__ uint8_t c_len_extra[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2,
                                        2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
__constant__ uint16_t c_dist_base[30] = {1,    2,    3,    4,    5,    7,     9,     13,    17,  25,
                                         33,   49,   65,   97,   129,  193,   257,   385,   513, 769,
                                         1025, 1537, 2049, 3073, 4097, 6145,  8193,  12289, 16385, 24577};
__constant__ uint8_t c_dist_extra[30] = {0, 0, 0, 0, 1, 1, 2, 2,  3,  3,  4,  4,  5,  5,  6,
                                         6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};

struct Huff {
  int16_t count[16];    // codes of each length
  int16_t symbol[288];  // symbols in canonical order
};

// canonical tables from code lengths; < 0 if over-subscribed
__device__ int build_huff(Huff* h, const uint8_t* length, int n) {
  for (int l = 0; l < 16; ++l) h->count[l] = 0;
  for (int i = 0; i < n; ++i) h->count[length[i]]++;
  if (h->count[0] == n) return 0;
  int left = 1;
  for (int l = 1; l < 16; ++l) {
    left <<= 1;
    left -= h->count[l];
    if (left < 0) return -1;
  }
  int16_t offs[16];
  offs[1] = 0;
  for (int l = 1; l < 15; ++l) offs[l + 1] = offs[l] + h->count[l];
  for (int i = 0; i < n; ++i)
    if (length[i]) h->symbol[offs[length[i]]++] = (int16_t)i;
  return left;
}

struct BitIn {
  const uint8_t* p;
  const uint8_t* end;
  uint64_t buf;
  int cnt;
  int over;  // bytes read past the end (zeros)
};

__device__ __forceinline__ void refill(BitIn& s) {
  if (s.cnt <= 32 && s.p + 4 <= s.end) {  // four bytes at once (independent loads)
    const uint64_t w = (uint64_t)s.p[0] | ((uint64_t)s.p[1] << 8) | ((uint64_t)s.p[2] << 16) |
                       ((uint64_t)s.p[3] << 24);
    s.buf |= w << s.cnt;
    s.cnt += 32;
    s.p += 4;
  }
  while (s.cnt <= 56) {
    uint64_t b = 0;
    if (s.p < s.end) b = *s.p++;
    else ++s.over;
    s.buf |= b << s.cnt;
    s.cnt += 8;
  }
}
__device__ __forceinline__ uint32_t getbits(BitIn& s, int n) {
  if (s.cnt < n) refill(s);
  const uint32_t v = (uint32_t)(s.buf & ((1ull << n) - 1));
  s.buf >>= n;
  s.cnt -= n;
  return v;
}
// Huffman codes are packed MSB first: walk lengths 1..15
__device__ __forceinline__ int decode_sym(BitIn& s, const Huff* h) {
  if (s.cnt < 15) refill(s);
  uint64_t bits = s.buf;
  int code = 0, first = 0, index = 0;
  for (int len = 1; len < 16; ++len) {
    code |= (int)(bits & 1);
    bits >>= 1;
    const int count = h->count[len];
    if (code - count < first) {
      s.buf >>= len;
      s.cnt -= len;
      return h->symbol[index + (code - first)];
    }
    index += count;
    first += count;
    first <<= 1;
    code <<= 1;
  }
  return -1;
}

enum { kBad = 1, kShort = 2, kLong = 3, kAdler = 4, kHeader = 5 };

// One zlib stream -> out[0, out_len); returns 0 or an error code.
__device__ int inflate_one(const uint8_t* in, int64_t in_len, uint8_t* out, int64_t out_len,
                           Huff& lencode, Huff& distcode) {
  if (in_len < 2) return kHeader;
  const uint32_t cmf = in[0], flg = in[1];
  if ((cmf & 15) != 8 || (cmf >> 4) > 7 || ((cmf << 8) | flg) % 31 != 0 || (flg & 0x20)) return kHeader;
  BitIn s{in + 2, in + in_len, 0, 0, 0};
  uint8_t lengths[320];
  int64_t o = 0;
  int last;
  do {
    last = (int)getbits(s, 1);
    const int type = (int)getbits(s, 2);
    if (type == 0) {  // stored: to a byte boundary, LEN, NLEN, bytes
      const int drop = s.cnt & 7;
      s.buf >>= drop;
      s.cnt -= drop;
      const uint32_t len = getbits(s, 16), nlen = getbits(s, 16);
      if ((len ^ 0xFFFFu) != nlen) return kBad;
      if (o + len > out_len) return kLong;
      uint32_t k = 0;
      while (k < len && s.cnt >= 8) {  // bytes still in the bit buffer
        out[o++] = (uint8_t)s.buf;
        s.buf >>= 8;
        s.cnt -= 8;
        ++k;
      }
      if (s.p + (len - k) > s.end) return kShort;
      for (; k < len; ++k) out[o++] = *s.p++;
      continue;
    }
    if (type == 3) return kBad;
    if (type == 1) {
      for (int i = 0; i < 144; ++i) lengths[i] = 8;
      for (int i = 144; i < 256; ++i) lengths[i] = 9;
      for (int i = 256; i < 280; ++i) lengths[i] = 7;
      for (int i = 280; i < 288; ++i) lengths[i] = 8;
      build_huff(&lencode, lengths, 288);
      for (int i = 0; i < 30; ++i) lengths[i] = 5;
      build_huff(&distcode, lengths, 30);
    } else {
      const int nlen = (int)getbits(s, 5) + 257, ndist = (int)getbits(s, 5) + 1;
      const int ncode = (int)getbits(s, 4) + 4;
      if (nlen > 286 || ndist > 30) return kBad;
      const uint8_t order[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};
      for (int i = 0; i < 19; ++i) lengths[i] = 0;
      for (int i = 0; i < ncode; ++i) lengths[order[i]] = (uint8_t)getbits(s, 3);
      if (build_huff(&lencode, lengths, 19) != 0) return kBad;  // must be complete
      int i = 0;
      while (i < nlen + ndist) {
        int sym = decode_sym(s, &lencode);
        if (sym < 0) return kBad;
        if (sym < 16) {
          lengths[i++] = (uint8_t)sym;
          continue;
        }
        int len = 0, rep;
        if (sym == 16) {
          if (i == 0) return kBad;
          len = lengths[i - 1];
          rep = 3 + (int)getbits(s, 2);
        } else if (sym == 17) {
          rep = 3 + (int)getbits(s, 3);
        } else {
          rep = 11 + (int)getbits(s, 7);
        }
        if (i + rep > nlen + ndist) return kBad;
        while (rep--) lengths[i++] = (uint8_t)len;
      }
      if (lengths[256] == 0) return kBad;
      const int el = build_huff(&lencode, lengths, nlen);
      if (el < 0 || (el > 0 && nlen - lencode.count[0] != 1)) return kBad;
      const int ed = build_huff(&distcode, lengths + nlen, ndist);
      if (ed < 0 || (ed > 0 && ndist - distcode.count[0] != 1)) return kBad;
    }
    for (;;) {
      int sym = decode_sym(s, &lencode);
      if (sym < 0) return kBad;
      if (sym < 256) {
        if (o >= out_len) return kLong;
        out[o++] = (uint8_t)sym;
        continue;
      }
      if (sym == 256) break;
      sym -= 257;
      if (sym >= 29) return kBad;
      const int len = c_len_base[sym] + (int)getbits(s, c_len_extra[sym]);
      const int dsym = decode_sym(s, &distcode);
      if (dsym < 0 || dsym >= 30) return kBad;
      const int64_t dist = c_dist_base[dsym] + (int)getbits(s, c_dist_extra[dsym]);
      if (dist > o) return kBad;
      if (o + len > out_len) return kLong;
      const uint8_t* from = out + o - dist;
      for (int k = 0; k < len; ++k) out[o + k] = from[k];
      o += len;
    }
  } while (!last);
  if (o != out_len) return kShort;
  // Adler-32 trailer (big-endian) after the last block, byte aligned
  const int drop = s.cnt & 7;
  s.buf >>= drop;
  s.cnt -= drop;
  uint32_t want = 0;
  for (int k = 0; k < 4; ++k) want = (want << 8) | getbits(s, 8);
  if (s.over > 8) return kShort;
  uint32_t a = 1, b = 0;
  for (int64_t k = 0; k < out_len; ++k) {
    a += out[k];
    if (a >= 65521u) a -= 65521u;
    b += a;
    if (b >= 65521u) b -= 65521u;
  }
  return ((b << 16) | a) == want ? 0 : kAdler;
}


// ------------------------------------------------------- warp-wide inflate
// One warp per zlib stream.  All 32 lanes run the same (uniform) decode loop on
// the same bit buffer; what the warp buys is the memory side: the compressed
// bytes arrive as 128-byte blocks (one word per lane, the next block in
// flight) and are handed out by shuffle, the output lives in a 32 KB shared-
// memory window (the deflate history), Huffman codes of <= 9 bits resolve with
// one shared-memory lookup, matches are copied by all lanes, and the window is
// written to global memory in 8 KB pieces (with the Adler-32 sums) by all lanes.
constexpr int kWinBitsBig = 15;     // 32 KB window: the deflate history
constexpr int kWinBitsSmall = 13;   // 8 KB: streams that inflate to <= 8 KB (one-row strips) -- 2.4x the warps per SM
constexpr int kFlush = 8192;
constexpr int kLitBits = 11, kDistBits = 8;   // index bits of the litlen / distance lookup tables

struct WarpIn {
  const uint32_t* words;   // aligned words covering the stream
  int64_t nwords;          // words that hold stream bytes
  int64_t widx;            // next word to hand out
  uint32_t first_mask;     // keeps the stream's bytes of word 0
  uint32_t last_mask;      // ... and of the last word
  uint32_t cur, nxt;       // this lane's word of the current / next 128-byte block
  uint64_t buf;
  int cnt;
  int lane;
};

__device__ __forceinline__ uint32_t wi_load(const WarpIn& s, int64_t block) {
  const int64_t i = block * 32 + s.lane;
  if (i >= s.nwords) return 0u;
  uint32_t w = __ldg(s.words + i);
  if (i == 0) w &= s.first_mask;
  if (i == s.nwords - 1) w &= s.last_mask;
  return w;
}
__device__ __forceinline__ void wi_refill(WarpIn& s) {
  if (s.cnt <= 32) {
    const int k = (int)(s.widx & 31);
    if (k == 0 && s.widx > 0) {
      s.cur = s.nxt;
      s.nxt = wi_load(s, (s.widx >> 5) + 1);
    }
    const uint32_t w = __shfl_sync(0xffffffffu, s.cur, k);
    s.buf |= (uint64_t)w << s.cnt;
    s.cnt += 32;
    ++s.widx;
  }
}
__device__ __forceinline__ uint32_t wi_bits(WarpIn& s, int n) {
  wi_refill(s);
  const uint32_t v = (uint32_t)(s.buf & ((1ull << n) - 1));
  s.buf >>= n;
  s.cnt -= n;
  return v;
}
// canonical walk (codes longer than the fast table's index)
__device__ __forceinline__ int wi_slow_sym(WarpIn& s, const Huff* h) {
  uint64_t bits = s.buf;
  int code = 0, first = 0, index = 0;
  for (int len = 1; len < 16; ++len) {
    code |= (int)(bits & 1);
    bits >>= 1;
    const int count = h->count[len];
    if (code - count < first) {
      s.buf >>= len;
      s.cnt -= len;
      return h->symbol[index + (code - first)];
    }
    index += count;
    first += count;
    first <<= 1;
    code <<= 1;
  }
  return -1;
}
template <int BITS>
__device__ __forceinline__ int wi_sym(WarpIn& s, const Huff* h, const uint16_t* fast) {
  wi_refill(s);   // >= 32 bits: enough for a code (15) and its extra bits (13)
  const uint32_t e = fast[s.buf & ((1u << BITS) - 1)];
  if (e & 15u) {
    s.buf >>= (e & 15u);
    s.cnt -= (int)(e & 15u);
    return (int)(e >> 4);
  }
  return wi_slow_sym(s, h);
}
// fast[the next BITS stream bits] = symbol << 4 | code length (0: longer code)
template <int BITS>
__device__ void wi_build_fast(const Huff* h, uint16_t* fast, int lane) {
  constexpr int kFast = 1 << BITS;
  for (int j = lane; j < kFast; j += 32) fast[j] = 0;
  __syncwarp();
  int code = 0, idx = 0;
  for (int l = 1; l <= BITS; ++l) {
    const int cnt = h->count[l];
    for (int i = 0; i < cnt; ++i, ++idx, ++code) {
      const uint32_t rev = __brev((uint32_t)code) >> (32 - l);   // stream order: first code bit lowest
      const uint16_t e = (uint16_t)((h->symbol[idx] << 4) | l);
      for (int j = (int)rev + (lane << l); j < kFast; j += 32 << l) fast[j] = e;
    }
    code <<= 1;
  }
  __syncwarp();
}

// lit2[next kLitBits stream bits] = bits consumed | count << 5 | first literal << 8 |
// second literal << 16: the literal the bits start with and, if its code leaves room
// for another complete literal code, that one too (count 1 or 2); 0 if the bits start
// with a length / end-of-block symbol or a code longer than the table index.
__device__ void wi_build_lit2(const uint16_t* fast, uint32_t* lit2, int lane) {
  constexpr int kFast = 1 << kLitBits;
  for (int i = lane; i < kFast; i += 32) {
    const uint32_t e1 = fast[i], l1 = e1 & 15u, s1 = e1 >> 4;
    uint32_t v = 0u;
    if (l1 != 0u && s1 < 256u) {
      v = l1 | (1u << 5) | (s1 << 8);
      const uint32_t e2 = fast[(uint32_t)i >> l1], l2 = e2 & 15u, s2 = e2 >> 4;   // high bits read as 0
      if (l2 != 0u && l1 + l2 <= (uint32_t)kLitBits && s2 < 256u) v = (l1 + l2) | (2u << 5) | (s1 << 8) | (s2 << 16);
    }
    lit2[i] = v;
  }
  __syncwarp();
}

template <int WB>
struct WarpSmem {
  static constexpr int kWin = 1 << WB, kWinMask = kWin - 1;
  uint8_t win[kWin];
  uint16_t litfast[1 << kLitBits];
  uint16_t distfast[1 << kDistBits];
  uint32_t lit2[1 << kLitBits];   // one or two literals per lookup (see wi_build_lit2)
  Huff lencode, distcode;
  uint8_t lengths[320];
};

// Adler-32 of win[from, from + n) folded into (a, b); all lanes, n <= kFlush
template <int kWinMask>
__device__ __forceinline__ void wi_flush(const uint8_t* win, uint8_t* out, int64_t from, int n,
                                         uint32_t& a, uint32_t& b, int lane) {
  unsigned long long sa = 0, sb = 0;
  for (int k = lane; k < n; k += 32) {
    const uint32_t d = win[(from + k) & kWinMask];
    out[from + k] = (uint8_t)d;
    sa += d;
    sb += (unsigned long long)(n - k) * d;
  }
  for (int o = 16; o > 0; o >>= 1) {
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
  }
  b = (uint32_t)((b + (unsigned long long)n * a + sb) % 65521ull);
  a = (uint32_t)((a + sa) % 65521ull);
}

template <int WB>
__device__ int inflate_warp(const uint8_t* in, int64_t in_len, uint8_t* out, int64_t out_len,
                            WarpSmem<WB>& m, int lane) {
  constexpr int kWinMask = WarpSmem<WB>::kWinMask;
  if (WB < kWinBitsBig && out_len > WarpSmem<WB>::kWin) return kLong;   // caller's promise broken
  if (in_len < 2) return kHeader;
  const uint32_t cmf = in[0], flg = in[1];
  if ((cmf & 15) != 8 || (cmf >> 4) > 7 || ((cmf << 8) | flg) % 31 != 0 || (flg & 0x20)) return kHeader;
  WarpIn s;
  {
    const uintptr_t p0 = reinterpret_cast<uintptr_t>(in) + 2, p1 = reinterpret_cast<uintptr_t>(in) + in_len;
    const uintptr_t w0 = p0 & ~(uintptr_t)3;
    s.words = reinterpret_cast<const uint32_t*>(w0);
    s.nwords = (int64_t)((p1 - w0 + 3) >> 2);
    s.first_mask = 0xffffffffu << (8 * (p0 & 3));
    s.last_mask = (p1 & 3) ? (0xffffffffu >> (8 * (4 - (p1 & 3)))) : 0xffffffffu;
    s.widx = 0;
    s.buf = 0;
    s.cnt = 0;
    s.lane = lane;
    s.cur = wi_load(s, 0);
    s.nxt = wi_load(s, 1);
    wi_refill(s);
    const int skip = 8 * (int)(p0 & 3);   // bytes of word 0 before the stream
    s.buf >>= skip;
    s.cnt -= skip;
  }
  const int64_t in_bits = 8 * (in_len - 2);
  auto used_bits = [&]() { return s.widx * 32 - 8 * (int64_t)((reinterpret_cast<uintptr_t>(in) + 2) & 3) - s.cnt; };
  int64_t o = 0, flushed = 0;
  uint32_t a = 1, b = 0;
  int last;
  do {
    last = (int)wi_bits(s, 1);
    const int type = (int)wi_bits(s, 2);
    if (type == 0) {  // stored: to a byte boundary, LEN, NLEN, bytes
      const int drop = s.cnt & 7;
      s.buf >>= drop;
      s.cnt -= drop;
      const uint32_t len = wi_bits(s, 16), nlen = wi_bits(s, 16);
      if ((len ^ 0xFFFFu) != nlen) return kBad;
      if (o + len > out_len) return kLong;
      for (uint32_t k = 0; k < len; ++k) {
        const uint32_t v = wi_bits(s, 8);
        if (lane == 0) m.win[(o + k) & kWinMask] = (uint8_t)v;
        if (((o + k + 1) & (kFlush - 1)) == 0) {
          __syncwarp();
          wi_flush<kWinMask>(m.win, out, flushed, kFlush, a, b, lane);
          flushed += kFlush;
        }
      }
      o += len;
      if (used_bits() > in_bits) return kShort;
      continue;
    }
    if (type == 3) return kBad;
    __syncwarp();
    if (type == 1) {
      for (int i = lane; i < 288; i += 32) m.lengths[i] = i < 144 ? 8 : i < 256 ? 9 : i < 280 ? 7 : 8;
      __syncwarp();
      if (lane == 0) build_huff(&m.lencode, m.lengths, 288);
      __syncwarp();
      for (int i = lane; i < 30; i += 32) m.lengths[i] = 5;
      __syncwarp();
      if (lane == 0) build_huff(&m.distcode, m.lengths, 30);
      __syncwarp();
    } else {
      const int nlen = (int)wi_bits(s, 5) + 257, ndist = (int)wi_bits(s, 5) + 1;
      const int ncode = (int)wi_bits(s, 4) + 4;
      if (nlen > 286 || ndist > 30) return kBad;
      const uint8_t order[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};
      if (lane < 19) m.lengths[lane] = 0;
      __syncwarp();
      for (int i = 0; i < ncode; ++i) {
        const uint32_t v = wi_bits(s, 3);
        if (lane == 0) m.lengths[order[i]] = (uint8_t)v;
      }
      __syncwarp();
      int rc = 0;
      if (lane == 0) rc = build_huff(&m.lencode, m.lengths, 19);
      rc = __shfl_sync(0xffffffffu, rc, 0);
      if (rc != 0) return kBad;  // must be complete
      __syncwarp();
      int i = 0;
      int prev_len = 0;
      while (i < nlen + ndist) {
        wi_refill(s);
        const int sym = wi_slow_sym(s, &m.lencode);
        if (sym < 0) return kBad;
        if (sym < 16) {
          if (lane == 0) m.lengths[i] = (uint8_t)sym;
          prev_len = sym;
          ++i;
          continue;
        }
        int len = 0, rep;
        if (sym == 16) {
          if (i == 0) return kBad;
          len = prev_len;
          rep = 3 + (int)wi_bits(s, 2);
        } else if (sym == 17) {
          rep = 3 + (int)wi_bits(s, 3);
        } else {
          rep = 11 + (int)wi_bits(s, 7);
        }
        if (i + rep > nlen + ndist) return kBad;
        for (int k = lane; k < rep; k += 32) m.lengths[i + k] = (uint8_t)len;
        prev_len = len;
        i += rep;
      }
      __syncwarp();
      if (m.lengths[256] == 0) return kBad;
      int el = 0, ed = 0, ok = 1;
      if (lane == 0) {
        el = build_huff(&m.lencode, m.lengths, nlen);
        if (el < 0 || (el > 0 && nlen - m.lencode.count[0] != 1)) ok = 0;
        ed = build_huff(&m.distcode, m.lengths + nlen, ndist);
        if (ed < 0 || (ed > 0 && ndist - m.distcode.count[0] != 1)) ok = 0;
      }
      ok = __shfl_sync(0xffffffffu, ok, 0);
      if (!ok) return kBad;
      __syncwarp();
    }
    wi_build_fast<kLitBits>(&m.lencode, m.litfast, lane);
    wi_build_fast<kDistBits>(&m.distcode, m.distfast, lane);
    wi_build_lit2(m.litfast, m.lit2, lane);
    for (;;) {
      {  // literal run: one table lookup per literal up to the next flush boundary
        // (32-bit counters; every lane stores the same byte, so nothing diverges).
        // ncu of a PNG stream: the loop is bound by its taken branches and by the
        // shared-window base ptxas rebuilds (S2UR -> ULEA) in front of every lookup,
        // so three lookups are decoded per refill check -- topped up to >= 33 bits =
        // three table codes of <= 11 bits -- and the table
        // / window addresses live in registers the compiler cannot see through.
        const int64_t stop = flushed + kFlush < out_len ? flushed + kFlush : out_len;
        uint32_t left = stop > o ? (uint32_t)(stop - o) : 0u;
        uint32_t pos = (uint32_t)o & kWinMask;
        const uint32_t left0 = left;
        uint32_t lit_at, win_at;
        asm volatile("mov.u32 %0, %1;" : "=r"(lit_at) : "r"(smem_u32(m.lit2)));
        asm volatile("mov.u32 %0, %1;" : "=r"(win_at) : "r"(smem_u32(m.win)));
        // one lookup = one or two literals (<= kLitBits bits), or false (other symbol / long code)
        auto literal = [&]() -> bool {
          uint32_t e;
          asm volatile("ld.shared.u32 %0, [%1];"
                       : "=r"(e)
                       : "r"(lit_at + (((uint32_t)s.buf & ((1u << kLitBits) - 1)) << 2)));
          const uint32_t n = (e >> 5) & 3u, l = e & 31u;
          if (n == 0u) return false;
          asm volatile("st.shared.u8 [%0], %1;" ::"r"(win_at + pos), "r"((e >> 8) & 0xffu) : "memory");
          pos = (pos + 1u) & kWinMask;
          asm volatile(
              "{\n\t.reg .pred p;\n\t"
              "setp.eq.u32 p, %2, 2;\n\t"
              "@p st.shared.u8 [%0], %1;\n\t"
              "}" ::"r"(win_at + pos),
              "r"(e >> 16), "r"(n)
              : "memory");
          pos = (pos + n - 1u) & kWinMask;
          left -= n;
          s.buf >>= l;
          s.cnt -= (int)l;
          return true;
        };
        while (left >= 6u) {   // three lookups (<= 33 bits, <= 6 literals) per refill check
          wi_refill(s);
          wi_refill(s);          // a refill of an empty buffer leaves 32 bits: top it up to >= 33
          if (!literal()) break;
          if (!literal()) break;
          if (!literal()) break;
        }
        while (left >= 2u) {
          wi_refill(s);
          if (!literal()) break;
        }
        o += left0 - left;
      }
      int sym = wi_sym<kLitBits>(s, &m.lencode, m.litfast);
      if (sym < 0) return kBad;
      if (sym < 256) {
        if (o >= out_len) return kLong;
        if (lane == 0) m.win[o & kWinMask] = (uint8_t)sym;
        ++o;
      } else {
        if (sym == 256) break;
        sym -= 257;
        if (sym >= 29) return kBad;
        const int len = c_len_base[sym] + (int)wi_bits(s, c_len_extra[sym]);
        const int dsym = wi_sym<kDistBits>(s, &m.distcode, m.distfast);
        if (dsym < 0 || dsym >= 30) return kBad;
        const int64_t dist = c_dist_base[dsym] + (int)wi_bits(s, c_dist_extra[dsym]);
        if (dist > o) return kBad;
        if (o + len > out_len) return kLong;
        __syncwarp();   // the literals and matches so far are visible to every lane
        const int64_t from = o - dist;
        // a far match may read the window slots this copy overwrites (distance
        // close to the window size): every lane loads before any lane stores
        for (int k0 = 0; k0 < len; k0 += 32) {
          const int k = k0 + lane;
          uint8_t v = 0;
          if (k < len) v = m.win[(from + (dist >= len ? k : k % (int)dist)) & kWinMask];
          __syncwarp();
          if (k < len) m.win[(o + k) & kWinMask] = v;
        }
        o += len;
      }
      if (o - flushed >= kFlush) {
        __syncwarp();
        wi_flush<kWinMask>(m.win, out, flushed, kFlush, a, b, lane);
        flushed += kFlush;
        __syncwarp();
      }
    }
    if (used_bits() > in_bits) return kShort;
  } while (!last);
  if (o != out_len) return kShort;
  __syncwarp();
  while (flushed < o) {
    const int n = (int)((o - flushed) < kFlush ? (o - flushed) : kFlush);
    wi_flush<kWinMask>(m.win, out, flushed, n, a, b, lane);
    flushed += n;
  }
  // Adler-32 trailer (big-endian) after the last block, byte aligned
  const int drop = s.cnt & 7;
  s.buf >>= drop;
  s.cnt -= drop;
  uint32_t want = 0;
  for (int k = 0; k < 4; ++k) want = (want << 8) | wi_bits(s, 8);
  if (used_bits() > in_bits + 64) return kShort;
  return ((b << 16) | a) == want ? 0 : kAdler;
}

template <int WB>
__global__ void __launch_bounds__(32) inflate_warp_kernel(const uint8_t* __restrict__ src, const int64_t* in_off,
                                                          const int64_t* in_len, uint8_t* dst,
                                                          const int64_t* out_off, const int64_t* out_len,
                                                          int32_t* status) {
  __shared__ __align__(16) WarpSmem<WB> m;   // static (46.6 / 22 KB): table and window addresses are compile-time offsets
  const int64_t i = blockIdx.x;
  const int rc = inflate_warp(src + in_off[i], in_len[i], dst + out_off[i], out_len[i], m, (int)threadIdx.x);
  if (threadIdx.x == 0) status[i] = rc;
}

// one thread per stream; its Huffman tables live in shared memory (the
// decode loop reads them once per code bit)
constexpr int kInfThreads = 32;
__global__ void __launch_bounds__(kInfThreads) inflate_kernel(const uint8_t* __restrict__ src,
                                                              const int64_t* in_off, const int64_t* in_len,
                                                              int64_t n, uint8_t* dst, const int64_t* out_off,
                                                              const int64_t* out_len, int32_t* status) {
  __shared__ Huff tabs[2][kInfThreads];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  status[i] = inflate_one(src + in_off[i], in_len[i], dst + out_off[i], out_len[i],
                          tabs[0][threadIdx.x], tabs[1][threadIdx.x]);
}

__global__ void __launch_bounds__(256) strips_copy_kernel(const uint8_t* __restrict__ src, const int64_t* in_off,
                                                          const int64_t* in_len, uint8_t* dst,
                                                          const int64_t* out_off, const int64_t* out_len,
                                                          int32_t* status) {
  const int64_t i = blockIdx.x;
  const int64_t n = out_len[i];
  if (threadIdx.x == 0) status[i] = in_len[i] < n ? kShort : 0;
  const uint8_t* s = src + in_off[i];
  uint8_t* d = dst + out_off[i];
  const int64_t m = in_len[i] < n ? in_len[i] : n;
  if (((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d)) & 15) == 0) {
    const int64_t v = m >> 4;
    for (int64_t k = threadIdx.x; k < v; k += blockDim.x)
      reinterpret_cast<uint4*>(d)[k] = reinterpret_cast<const uint4*>(s)[k];
    for (int64_t k = (v << 4) + threadIdx.x; k < m; k += blockDim.x) d[k] = s[k];
  } else {
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) d[k] = s[k];
  }
}


// ------------------------------------------------------------------ TIFF LZW
// One LZW stream -> out[0, out_len).  pos / len: per-code string position and
// length in `out` (codes >= 258).
__device__ int lzw_one(const uint8_t* in, int64_t in_len, uint8_t* out, int64_t out_len,
                       int32_t* pos, uint16_t* len) {
  uint64_t buf = 0;   // MSB-first: the next code sits in the top bits
  int cnt = 0;
  int64_t ip = 0, o = 0;
  int width = 9, next = 258, prev = -1;
  int64_t prev_at = 0;
  int prev_len = 0;
  for (;;) {
    while (cnt <= 56 && ip < in_len) {
      buf |= (uint64_t)in[ip++] << (56 - cnt);
      cnt += 8;
    }
    if (cnt < width) break;                    // data ended without EOI: accepted if complete
    const int code = (int)(buf >> (64 - width));
    buf <<= width;
    cnt -= width;
    if (code == 257) break;                    // EOI
    if (code == 256) {                         // Clear
      width = 9;
      next = 258;
      prev = -1;
      continue;
    }
    int64_t at;
    int n;
    if (code < 256) {
      if (o >= out_len) return kLong;
      at = o;
      n = 1;
      out[o++] = (uint8_t)code;
    } else {
      if (prev < 0) return kBad;
      int64_t from;
      if (code < next) {
        from = pos[code];
        n = len[code];
      } else if (code == next) {               // KwKwK: previous string + its first byte
        from = prev_at;
        n = prev_len + 1;
      } else {
        return kBad;
      }
      if (o + n > out_len) return kLong;
      at = o;
      for (int k = 0; k < n; ++k) out[o + k] = out[from + k];
      o += n;
    }
    if (prev >= 0 && next < 4096) {            // new entry: previous string + first byte of this one
      if (prev_len + 1 > 65535) return kBad;
      pos[next] = (int32_t)prev_at;
      len[next] = (uint16_t)(prev_len + 1);
      ++next;
    }
    prev = code;
    prev_at = at;
    prev_len = n;
    // early change: the width grows one code before the table fills the current width
    if (next + 1 >= (1 << width) && width < 12) ++width;
  }
  return o == out_len ? 0 : kShort;
}

constexpr int kLzwThreads = 32;
__global__ void __launch_bounds__(kLzwThreads) lzw_kernel(const uint8_t* __restrict__ src, const int64_t* in_off,
                                                          const int64_t* in_len, int64_t n, uint8_t* dst,
                                                          const int64_t* out_off, const int64_t* out_len,
                                                          int32_t* status, int32_t* pos_ws, uint16_t* len_ws) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  status[i] = out_len[i] >= ((int64_t)1 << 31)
                  ? kLong
                  : lzw_one(src + in_off[i], in_len[i], dst + out_off[i], out_len[i], pos_ws + i * 4096,
                            len_ws + i * 4096);
}

// ------------------------------------------------------------------ tiles
// tile t = (ty, tx) holds tile_rows x tile_row_bytes bytes; the image gets the part inside it
__global__ void __launch_bounds__(256) untile_kernel(const uint8_t* __restrict__ tiles, uint8_t* __restrict__ img,
                                                     int64_t rows, int64_t row_bytes, int64_t tile_rows,
                                                     int64_t tile_row_bytes, int64_t across) {
  const int64_t t = blockIdx.x, ty = t / across, tx = t - ty * across;
  const uint8_t* src = tiles + t * tile_rows * tile_row_bytes;
  const int64_t y0 = ty * tile_rows, b0 = tx * tile_row_bytes;
  const int64_t nr = rows - y0 < tile_rows ? rows - y0 : tile_rows;
  const int64_t nb = row_bytes - b0 < tile_row_bytes ? row_bytes - b0 : tile_row_bytes;
  for (int64_t e = threadIdx.x; e < nr * nb; e += blockDim.x) {
    const int64_t r = e / nb, c = e - r * nb;
    img[(y0 + r) * row_bytes + b0 + c] = src[r * tile_row_bytes + c];
  }
}

// ------------------------------------------------------------------ PNG filters
constexpr int kPngCx = 32;        // pixel columns per staged chunk (>= 32: the wavefront spans two chunks)
constexpr int kPngMaxBpp = 8;

__device__ __forceinline__ uint32_t paeth(uint32_t a, uint32_t b, uint32_t c) {
  const int pa = abs((int)b - (int)c), pb = abs((int)a - (int)c), pc = abs((int)a + (int)b - 2 * (int)c);
  return (pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c);
}

// One image, BPP bytes per pixel (1: gray 8, 2: gray 16, 3: RGB 8, 6: RGB 16).  work holds
// the inflated scanlines ([filter byte][row bytes] per row); they are reconstructed
// in place by one warp.
template <int BPP>
__device__ int png_unfilter_image(uint8_t* __restrict__ base, int64_t rows, int64_t cols,
                                  uint8_t (*sin)[33][kPngCx * kPngMaxBpp],
                                  uint8_t (*sout)[32][kPngCx * kPngMaxBpp], int lane) {
  constexpr int CB = kPngCx * BPP;           // bytes of a full chunk row
  constexpr int IT = (CB + 31) / 32;         // byte loads per lane and row
  const int64_t rb = cols * BPP, stride = rb + 1;
  const int64_t nchunks = (cols + kPngCx - 1) / kPngCx;
  int bad = 0;
  for (int64_t y0 = 0; y0 < rows; y0 += 32) {
    const int64_t y = y0 + lane;
    const bool live = y < rows;
    const int ft = live ? base[y * stride] : 0;
    if (ft > 4) bad = 1;
    uint32_t a[BPP], b[BPP], c[BPP];
#pragma unroll
    for (int j = 0; j < BPP; ++j) a[j] = b[j] = c[j] = 0;
    // filtered bytes of chunk k of the 32 rows + the row above: four rows' loads are
    // issued together (one memory latency per four rows, not per row)
    auto load_chunk = [&](int64_t k) {
      const int buf = (int)(k & 1);
      const int64_t c0 = k * CB;
      const int nb = (int)((rb - c0) < (int64_t)CB ? (rb - c0) : (int64_t)CB);
      for (int r0 = 0; r0 < 33; r0 += 4) {
        uint8_t v[4][IT];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = r0 + q;
          const int64_t yy = r < 32 ? y0 + r : y0 - 1;
          const bool ok = r < 33 && yy >= 0 && yy < rows;
          const uint8_t* src = base + (ok ? yy : 0) * stride + 1 + c0;
#pragma unroll
          for (int it = 0; it < IT; ++it) {
            const int e = it * 32 + lane;
            v[q][it] = (ok && e < nb) ? src[e] : (uint8_t)0;
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = r0 + q;
          if (r < 33) {
#pragma unroll
            for (int it = 0; it < IT; ++it) {
              const int e = it * 32 + lane;
              if (e < CB) sin[buf][r][e] = v[q][it];
            }
          }
        }
      }
    };
    auto flush_chunk = [&](int64_t k) {  // reconstructed bytes of chunk k back in place
      const int buf = (int)(k & 1);
      const int64_t c0 = k * CB;
      const int nb = (int)((rb - c0) < (int64_t)CB ? (rb - c0) : (int64_t)CB);
      for (int r = 0; r < 32 && y0 + r < rows; ++r) {
        uint8_t* dst = base + (y0 + r) * stride + 1 + c0;
        for (int e = lane; e < nb; e += 32) dst[e] = sout[buf][r][e];
      }
    };
    const int64_t steps = cols + 31;
    for (int64_t s = 0; s < steps; ++s) {
      if (s % kPngCx == 0) {
        const int64_t k = s / kPngCx;
        __syncwarp();
        if (k >= 2) flush_chunk(k - 2);
        if (k < nchunks) load_chunk(k);
        __syncwarp();
      }
      // the pixel lane - 1 produced last step is this lane's "up" pixel
      uint32_t up[BPP];
#pragma unroll
      for (int j = 0; j < BPP; ++j) up[j] = __shfl_up_sync(0xffffffffu, a[j], 1);
      const int64_t x = s - lane;
      if (live && x >= 0 && x < cols) {
        const int buf = (int)((x / kPngCx) & 1);
        const int xc = (int)(x % kPngCx) * BPP;
#pragma unroll
        for (int j = 0; j < BPP; ++j) {
          c[j] = x == 0 ? 0u : b[j];
          b[j] = lane == 0 ? (uint32_t)sin[buf][32][xc + j] : up[j];
          const uint32_t left = x == 0 ? 0u : a[j];
          uint32_t pred = 0;
          if (ft == 1) pred = left;
          else if (ft == 2) pred = b[j];
          else if (ft == 3) pred = (left + b[j]) >> 1;
          else if (ft == 4) pred = paeth(left, b[j], c[j]);
          a[j] = ((uint32_t)sin[buf][lane][xc + j] + pred) & 0xffu;
          sout[buf][lane][xc + j] = (uint8_t)a[j];
        }
      }
    }
    __syncwarp();
    if (nchunks >= 2) flush_chunk(nchunks - 2);
    flush_chunk(nchunks - 1);
    __syncwarp();
    __threadfence_block();
  }
  return __any_sync(0xffffffffu, bad);
}

// table row i: work_off, out_off, rows, cols, channels, depth.  One warp per image.
__global__ void __launch_bounds__(32) png_unfilter_kernel(uint8_t* __restrict__ work,
                                                          const int64_t* __restrict__ table,
                                                          int32_t* __restrict__ status) {
  __shared__ uint8_t sin[2][33][kPngCx * kPngMaxBpp];   // row 32 = the row above the group
  __shared__ uint8_t sout[2][32][kPngCx * kPngMaxBpp];
  const int64_t* tb = table + (int64_t)blockIdx.x * 6;
  const int64_t rows = tb[2], cols = tb[3];
  const int bpp = (int)(tb[4] * tb[5] / 8);
  uint8_t* base = work + tb[0];
  const int lane = threadIdx.x;
  int bad;
  switch (bpp) {
    case 1: bad = png_unfilter_image<1>(base, rows, cols, sin, sout, lane); break;
    case 2: bad = png_unfilter_image<2>(base, rows, cols, sin, sout, lane); break;
    case 3: bad = png_unfilter_image<3>(base, rows, cols, sin, sout, lane); break;
    case 6: bad = png_unfilter_image<6>(base, rows, cols, sin, sout, lane); break;
    default: bad = 1; break;
  }
  if (lane == 0) status[blockIdx.x] = bad ? kBad : 0;
}

// reconstructed scanlines -> image rows (filter byte dropped, 16-bit samples to little endian)
__global__ void __launch_bounds__(256) png_rows_kernel(const uint8_t* __restrict__ work,
                                                       const int64_t* __restrict__ table,
                                                       uint8_t* __restrict__ out) {
  const int64_t* tb = table + (int64_t)blockIdx.y * 6;
  const int64_t rows = tb[2], cols = tb[3];
  const int bpp = (int)(tb[4] * tb[5] / 8);
  const bool swap = tb[5] == 16;
  const int64_t rb = cols * bpp, stride = rb + 1;
  const uint8_t* base = work + tb[0];
  uint8_t* dst = out + tb[1];
  for (int64_t y = blockIdx.x; y < rows; y += gridDim.x) {
    const uint8_t* src = base + y * stride + 1;
    uint8_t* d = dst + y * rb;
    for (int64_t e = threadIdx.x; e < rb; e += blockDim.x) d[e] = src[swap ? (e ^ 1) : e];
  }
}

// One warp per row: a chunk of the row per step (32 samples, or 30 for RGB so that
// a chunk holds whole pixels), the running sums of Predictor 2 by a shuffle scan
// along each channel's chain (offsets ch, 2 ch, 4 ch, ...) plus the carry of the
// previous chunk -- coalesced accesses and 32x the threads of a thread per row.
template <typename T>
__global__ void __launch_bounds__(128) unpredict_kernel(T* img, int64_t rows, int64_t spr, int ch,
                                                        int predictor, int swap) {
  const int lane = threadIdx.x & 31;
  const int64_t y = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (y >= rows) return;   // warp-uniform
  T* row = img + y * spr;
  const int chunk = 32 - (32 % ch);
  const int tail = chunk - ch + lane % ch;   // lane holding this lane's channel at the chunk's end
  uint32_t carry = 0u;
  for (int64_t x0 = 0; x0 < spr; x0 += chunk) {
    const int64_t x = x0 + lane;
    const bool active = lane < chunk && x < spr;
    uint32_t v = active ? (uint32_t)row[x] : 0u;
    if (swap && sizeof(T) == 2) v = ((v >> 8) | (v << 8)) & 0xffffu;
    if (predictor == 2) {
      for (int o = ch; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
      }
      v += carry;
      carry = __shfl_sync(0xffffffffu, v, tail);
    }
    if (active) row[x] = (T)v;
  }
}

}  // namespace
}  // namespace ut

using namespace ut;

extern "C" {

int ut_decode_strips(const uint8_t* src, const int64_t* in_off, const int64_t* in_len, int64_t nstrips,
                     int32_t compression, uint8_t* dst, const int64_t* out_off, const int64_t* out_len,
                     int32_t* status, void* stream) {
  return ut_decode_streams(src, in_off, in_len, nstrips, compression, dst, out_off, out_len, 0, status,
                           stream);
}

int ut_decode_streams(const uint8_t* src, const int64_t* in_off, const int64_t* in_len, int64_t nstrips,
                      int32_t compression, uint8_t* dst, const int64_t* out_off, const int64_t* out_len,
                      int64_t max_out_len, int32_t* status, void* stream) {
  UT_REQUIRE(nstrips >= 0, "negative strip count");
  UT_REQUIRE(compression == 1 || compression == 8 || compression == 5,
             "strip compression must be 1 (none), 5 (LZW) or 8 (zlib deflate), got %d", compression);
  if (nstrips == 0) return UT_OK;
  UT_REQUIRE(src && in_off && in_len && dst && out_off && out_len && status, "ut_decode_strips: null pointer");
  cudaStream_t st = as_stream(stream);
  if (compression == 1) {
    strips_copy_kernel<<<(unsigned)nstrips, 256, 0, st>>>(src, in_off, in_len, dst, out_off, out_len, status);
    UT_CHECK_LAUNCH("strips_copy_kernel");
  } else if (compression == 5) {
    // string tables: 6 bytes per code and stream in a stream-ordered scratch buffer;
    // at most 32768 streams (768 MB of tables) per launch, so a stack of many one-row
    // strips does not ask for tens of gigabytes
    constexpr int64_t kWave = 32768;
    const int64_t wave = nstrips < kWave ? nstrips : kWave;
    void* tab = nullptr;
    const size_t per = 4096 * (sizeof(int32_t) + sizeof(uint16_t));
    cudaError_t e = cudaMallocAsync(&tab, per * (size_t)wave, st);
    if (e != cudaSuccess) return cuda_status(e, "ut_decode_strips: LZW tables");
    int32_t* pos = static_cast<int32_t*>(tab);
    uint16_t* len = reinterpret_cast<uint16_t*>(pos + (size_t)wave * 4096);
    cudaError_t le = cudaSuccess;
    for (int64_t s0 = 0; s0 < nstrips && le == cudaSuccess; s0 += wave) {
      const int64_t n = nstrips - s0 < wave ? nstrips - s0 : wave;
      lzw_kernel<<<(unsigned)((n + kLzwThreads - 1) / kLzwThreads), kLzwThreads, 0, st>>>(
          src, in_off + s0, in_len + s0, n, dst, out_off + s0, out_len + s0, status + s0, pos, len);
      le = cudaGetLastError();
    }
    cudaFreeAsync(tab, st);
    if (le != cudaSuccess) return cuda_status(le, "lzw_kernel");
  } else {
    static const bool thread_mode = [] {
      const char* e = getenv("UT_INFLATE_THREAD");   // dev: the one-thread-per-stream decoder
      return e && e[0] == '1';
    }();
    if (thread_mode) {
      inflate_kernel<<<(unsigned)((nstrips + kInfThreads - 1) / kInfThreads), kInfThreads, 0, st>>>(
          src, in_off, in_len, nstrips, dst, out_off, out_len, status);
      UT_CHECK_LAUNCH("inflate_kernel");
    } else {
      static_assert(sizeof(WarpSmem<kWinBitsBig>) <= 48 * 1024,
                    "inflate window + tables must fit static shared memory");
      // streams known to inflate to <= 8 KB each (e.g. one-row strips) take the
      // small-window kernel: 22 KB of shared memory per warp instead of 46.6 KB
      if (max_out_len > 0 && max_out_len <= (1 << kWinBitsSmall))
        inflate_warp_kernel<kWinBitsSmall><<<(unsigned)nstrips, 32, 0, st>>>(src, in_off, in_len, dst, out_off,
                                                                             out_len, status);
      else
        inflate_warp_kernel<kWinBitsBig><<<(unsigned)nstrips, 32, 0, st>>>(src, in_off, in_len, dst, out_off,
                                                                           out_len, status);
      UT_CHECK_LAUNCH("inflate_warp_kernel");
    }
  }
  return UT_OK;
}

int ut_unpredict(void* img, int32_t depth, int64_t rows, int64_t cols, int32_t channels, int32_t predictor,
                 int32_t swap_bytes, void* stream) {
  UT_REQUIRE(depth == 8 || depth == 16, "sample depth must be 8 or 16, got %d", depth);
  UT_REQUIRE(predictor == 1 || predictor == 2, "TIFF predictor must be 1 or 2, got %d", predictor);
  UT_REQUIRE(rows >= 0 && cols >= 0 && channels >= 1, "bad image geometry");
  if (rows == 0 || cols == 0 || (predictor == 1 && !(swap_bytes && depth == 16))) return UT_OK;
  cudaStream_t st = as_stream(stream);
  UT_REQUIRE(channels <= 16, "ut_unpredict: at most 16 channels");
  const unsigned grid = (unsigned)((rows * 32 + 127) / 128);   // one warp per row
  if (depth == 8)
    unpredict_kernel<uint8_t><<<grid, 128, 0, st>>>(static_cast<uint8_t*>(img), rows, cols * channels,
                                                    channels, predictor, 0);
  else
    unpredict_kernel<uint16_t><<<grid, 128, 0, st>>>(static_cast<uint16_t*>(img), rows, cols * channels,
                                                     channels, predictor, swap_bytes);
  UT_CHECK_LAUNCH("unpredict_kernel");
  return UT_OK;
}

int ut_untile(const uint8_t* tiles, uint8_t* img, int64_t rows, int64_t row_bytes, int64_t tile_rows,
              int64_t tile_row_bytes, int64_t tiles_across, int64_t ntiles, void* stream) {
  UT_REQUIRE(rows > 0 && row_bytes > 0 && tile_rows > 0 && tile_row_bytes > 0 && tiles_across > 0,
             "ut_untile: bad geometry");
  UT_REQUIRE(ntiles >= 0 && ntiles < ((int64_t)1 << 31), "ut_untile: bad tile count");
  if (ntiles == 0) return UT_OK;
  UT_REQUIRE(tiles && img, "ut_untile: null pointer");
  untile_kernel<<<(unsigned)ntiles, 256, 0, as_stream(stream)>>>(tiles, img, rows, row_bytes, tile_rows,
                                                                tile_row_bytes, tiles_across);
  UT_CHECK_LAUNCH("untile_kernel");
  return UT_OK;
}

int ut_png_unfilter(uint8_t* work, const int64_t* table, int64_t n, uint8_t* out, int32_t* status,
                    void* stream) {
  UT_REQUIRE(n >= 0 && n < 65536, "ut_png_unfilter: bad image count");
  if (n == 0) return UT_OK;
  UT_REQUIRE(work && table && out && status, "ut_png_unfilter: null pointer");
  cudaStream_t st = as_stream(stream);
  png_unfilter_kernel<<<(unsigned)n, 32, 0, st>>>(work, table, status);
  UT_CHECK_LAUNCH("png_unfilter_kernel");
  png_rows_kernel<<<dim3(64, (unsigned)n), 256, 0, st>>>(work, table, out);
  UT_CHECK_LAUNCH("png_rows_kernel");
  return UT_OK;
}

}  // extern "C"
