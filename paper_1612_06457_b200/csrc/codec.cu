// Image encoders of save_image (rendering.py:303-331): PNG (8/16-bit gray,
// 8-bit RGB) and TIFF (none / deflate), built from code planes resident in HBM.
//
// The reference hands the codes to cv2.imwrite (libpng / libtiff + zlib on one
// core).  Here the whole encode runs on the device and the host only writes
// the finished bytes:
//
//  * png_filter_kernel: PNG row filters (None/Sub/Up/Average/Paeth), chosen per
//    row by the minimum sum of |signed residual| (the libpng heuristic), 16-bit
//    samples big-endian.  tiff_predict_kernel: TIFF horizontal differencing
//    (Predictor 2) for deflate strips.
//  * deflate_kernel: one CTA per 32 KB "unit" of the filtered stream.  The unit
//    and up to 32 KB of history before it (same zlib stream) are staged in
//    shared memory; each thread parses a 128-byte sub-range greedily, testing a
//    fixed set of image-shaped match distances (1..4, the pixel, the row, the
//    row +- one pixel, two rows) and emitting fixed-Huffman literal / match
//    codes (RFC 1951 3.2.6).  Pass A counts bits, a block scan places every
//    thread's code, pass B writes it (shared-memory atomics at word seams).  A
//    unit closes with end-of-block + an empty stored block (a sync flush), so
//    every unit is byte-aligned and units concatenate.  A unit that would not
//    shrink is written as one stored block.  Per-unit Adler-32 parts ride along.
//  * deflate_frame_kernel: one CTA scans the unit sizes into final offsets and
//    writes the stream framing -- zlib header 78 01, the final empty block
//    03 00, Adler-32 (combined from the unit parts) -- for a PNG (one stream,
//    one IDAT chunk per unit) or a TIFF (one zlib stream per strip).
//  * deflate_place_kernel: one CTA per unit copies its bytes into place and,
//    for PNG, writes the chunk header and the chunk CRC-32 (per-thread CRCs
//    merged in a tree with the GF(2) shift operator x^(8n) mod P).
//
// Output is a pure function of the input bytes (no atomics whose order
// matters, fixed parse), so files are byte-deterministic (the reference's
// test_rendering.py:377-385 asks for that).
#include <algorithm>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace ut {
namespace {

constexpr int kUnit = 32768;                 // raw bytes per deflate unit
constexpr int kHist = 32768;                 // history window staged before a unit
constexpr int kDThreads = 256;
constexpr int kSub = kUnit / kDThreads;      // bytes parsed per thread
constexpr int kSlot = 32800;                 // >= stored form 5 + 32768, multiple of 16
constexpr int kMaxCand = 12;
constexpr uint32_t kAdlerMod = 65521u;
constexpr uint32_t kCrcPoly = 0xEDB88320u;   // reflected CRC-32 polynomial

__constant__ uint32_t c_x2n[32];             // x^(2^k) mod P (reflected), k = 0..31

// ------------------------------------------------------------------ CRC-32
__device__ __forceinline__ uint32_t multmodp(uint32_t a, uint32_t b) {
  uint32_t m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1)) == 0) break;
    }
    m >>= 1;
    b = (b & 1) ? (b >> 1) ^ kCrcPoly : b >> 1;
  }
  return p;
}
// x^(8 n) mod P: the operator that shifts a CRC past n zero bytes
__device__ __forceinline__ uint32_t x8nmodp(uint64_t n) {
  uint32_t p = 1u << 31;
  int k = 3;
  while (n) {
    if (n & 1) p = multmodp(c_x2n[k & 31], p);
    n >>= 1;
    ++k;
  }
  return p;
}
__device__ __forceinline__ uint32_t crc_bytes(const uint32_t* tab, uint32_t crc, const uint8_t* p,
                                              int64_t n) {
  crc = ~crc;
  for (int64_t i = 0; i < n; ++i) crc = tab[(crc ^ p[i]) & 0xFF] ^ (crc >> 8);
  return ~crc;
}
__device__ __forceinline__ void crc_table(uint32_t* tab) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t c = (uint32_t)i;
    for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ kCrcPoly : c >> 1;
    tab[i] = c;
  }
}

// -------------------------------------------------------------- PNG filters
__device__ __forceinline__ int png_byte(const uint8_t* row, int depth, int64_t k) {
  if (depth == 8) return row[k];
  const uint16_t v = reinterpret_cast<const uint16_t*>(row)[k >> 1];
  return (k & 1) ? (v & 0xFF) : (v >> 8);     // PNG stores 16-bit samples big-endian
}
__device__ __forceinline__ int paeth(int a, int b, int c) {
  const int p = a + b - c;
  const int pa = abs(p - a), pb = abs(p - b), pc = abs(p - c);
  if (pa <= pb && pa <= pc) return a;
  return pb <= pc ? b : c;
}
__device__ __forceinline__ int png_residual(int f, int x, int a, int b, int c) {
  switch (f) {
    case 0: return x;
    case 1: return (x - a) & 0xFF;
    case 2: return (x - b) & 0xFF;
    case 3: return (x - ((a + b) >> 1)) & 0xFF;
    default: return (x - paeth(a, b, c)) & 0xFF;
  }
}

// one CTA per image row: out row = [filter type][rb residual bytes]
__global__ void __launch_bounds__(256) png_filter_kernel(const uint8_t* __restrict__ img, int64_t rb,
                                                         int depth, int bpp, uint8_t* __restrict__ out) {
  const int64_t y = blockIdx.x;
  const uint8_t* cur = img + y * rb;
  const uint8_t* prev = y > 0 ? cur - rb : nullptr;
  uint32_t cost[5] = {0, 0, 0, 0, 0};
  for (int64_t k = threadIdx.x; k < rb; k += blockDim.x) {
    const int x = png_byte(cur, depth, k);
    const int a = k >= bpp ? png_byte(cur, depth, k - bpp) : 0;
    const int b = prev ? png_byte(prev, depth, k) : 0;
    const int c = (prev && k >= bpp) ? png_byte(prev, depth, k - bpp) : 0;
#pragma unroll
    for (int f = 0; f < 5; ++f) {
      const int r = png_residual(f, x, a, b, c);
      cost[f] += r < 128 ? r : 256 - r;        // |signed residual|
    }
  }
  __shared__ uint32_t red[5][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int f = 0; f < 5; ++f) {
    uint32_t v = cost[f];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[f][warp] = v;
  }
  __syncthreads();
  __shared__ int pick;
  if (threadIdx.x == 0) {
    uint64_t best = ~0ull;
    int bf = 0;
    for (int f = 0; f < 5; ++f) {
      uint64_t s = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[f][w];
      if (s < best) { best = s; bf = f; }    // ties keep the lower filter type
    }
    pick = bf;
  }
  __syncthreads();
  const int f = pick;
  uint8_t* o = out + y * (rb + 1);
  if (threadIdx.x == 0) o[0] = (uint8_t)f;
  for (int64_t k = threadIdx.x; k < rb; k += blockDim.x) {
    const int x = png_byte(cur, depth, k);
    const int a = k >= bpp ? png_byte(cur, depth, k - bpp) : 0;
    const int b = prev ? png_byte(prev, depth, k) : 0;
    const int c = (prev && k >= bpp) ? png_byte(prev, depth, k - bpp) : 0;
    o[1 + k] = (uint8_t)png_residual(f, x, a, b, c);
  }
}

// TIFF Predictor 2: each sample minus the same channel of the previous pixel
// (mod 2^depth), rows independent, samples in native (little-endian) order.
template <typename T>
__global__ void tiff_predict_kernel(const T* __restrict__ img, int64_t rows, int64_t spr /*samples per row*/,
                                    int ch, T* __restrict__ out) {
  const int64_t n = rows * spr;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = i % spr;
    out[i] = x >= ch ? (T)(img[i] - img[i - ch]) : img[i];
  }
}

// ------------------------------------------------------------------ deflate
struct DeflateParams {
  const uint8_t* data;   // filtered bytes, streams back to back
  int64_t stream_len;    // bytes per stream (all but the last)
  int64_t last_len;      // bytes of the last stream
  int32_t nstreams;
  int32_t upc;           // units per full stream
  int32_t nunits;
  int32_t ncand;
  int32_t cand[kMaxCand];  // candidate match distances, ascending, <= 32768
  uint8_t* slots;        // [nunits][kSlot]
  int32_t* ulen;         // bytes of each unit's deflate output
  uint32_t* uadler;      // [nunits][2]: sum b_i, sum (len - i) b_i  (mod 65521)
};

struct UnitGeom {
  int stream;
  int64_t start;         // first byte of the unit in `data`
  int64_t off;           // offset of the unit inside its stream
  int len, hist;
};
__device__ __forceinline__ UnitGeom unit_geom(int64_t stream_len, int64_t last_len, int nstreams,
                                              int upc, int u) {
  UnitGeom g;
  g.stream = u / upc;
  const int idx = u - g.stream * upc;
  const int64_t slen = g.stream == nstreams - 1 ? last_len : stream_len;
  g.off = (int64_t)idx * kUnit;
  g.start = (int64_t)g.stream * stream_len + g.off;
  g.len = (int)(int)(slen - g.off < kUnit ? slen - g.off : kUnit);
  g.hist = (int)(g.off < kHist ? g.off : kHist);
  return g;
}

__device__ __forceinline__ uint32_t rev_bits(uint32_t code, int n) { return __brev(code) >> (32 - n); }

// fixed-Huffman literal/length code of symbol s (0..287), bit-reversed for the
// LSB-first stream; returns the code length
__device__ __forceinline__ int litlen_code(int s, uint32_t* code) {
  if (s < 144) { *code = rev_bits(0x30 + s, 8); return 8; }
  if (s < 256) { *code = rev_bits(0x190 + (s - 144), 9); return 9; }
  if (s < 280) { *code = rev_bits(s - 256, 7); return 7; }
  *code = rev_bits(0xC0 + (s - 280), 8);
  return 8;
}
// length 3..258 -> symbol, extra bit count, extra value
__device__ __forceinline__ void length_sym(int L, int* sym, int* nx, int* xv) {
  const int x = L - 3;
  if (L == 258) { *sym = 285; *nx = 0; *xv = 0; return; }
  if (x < 8) { *sym = 257 + x; *nx = 0; *xv = 0; return; }
  const int k = 31 - __clz(x);
  const int hi = (x >> (k - 2)) & 3;
  *sym = 257 + 4 * (k - 1) + hi;
  *nx = k - 2;
  *xv = L - ((((4 + hi) << (k - 2))) + 3);
}
// distance 1..32768 -> symbol, extra bit count, extra value
__device__ __forceinline__ void dist_sym(int d, int* sym, int* nx, int* xv) {
  const int x = d - 1;
  if (x < 4) { *sym = x; *nx = 0; *xv = 0; return; }
  const int k = 31 - __clz(x);
  const int hi = (x >> (k - 1)) & 1;
  *sym = 2 * k + hi;
  *nx = k - 1;
  *xv = d - (((2 + hi) << (k - 1)) + 1);
}

__device__ __forceinline__ void put_bits(uint32_t* words, uint32_t& pos, uint32_t v, int n) {
  if (n == 0) return;
  const uint32_t w = pos >> 5, o = pos & 31;
  if (v) {
    atomicOr(&words[w], v << o);
    if (o + n > 32) atomicOr(&words[w + 1], v >> (32 - o));
  }
  pos += n;
}

// Per-unit code tables (shared memory).  Codes are stored bit-reversed for the
// LSB-first stream.
struct Codes {
  uint32_t lf[288], df[32];          // symbol frequencies (pass A)
  uint16_t lcode[288], dcode[32];
  uint8_t llen[288], dlen[32];
  uint32_t A[288];                   // Huffman build scratch
  uint16_t sym[288];
  uint32_t cf[19];                   // code-length alphabet
  uint16_t ccode[19];
  uint8_t clen[19];
  uint16_t rle[320];                 // code-length symbols: sym | extra << 5
  int nrle, hlit, hdist, hclen;
  uint32_t header_bits;
};

// histogram add aggregated over the lanes of the warp that are here with the
// same symbol (the parse loops diverge; hot symbols would serialize otherwise)
__device__ __forceinline__ void hist_add(uint32_t* h, int sym) {
  const unsigned mask = __match_any_sync(__activemask(), sym);
  if ((threadIdx.x & 31) == __ffs(mask) - 1) atomicAdd(&h[sym], (uint32_t)__popc(mask));
}

__device__ __forceinline__ int fixed_litlen_len(int s) {
  return s < 144 ? 8 : (s < 256 ? 9 : (s < 280 ? 7 : 8));
}

// Greedy parse of buf[base + q0 .. base + q1) (matches stay inside the range,
// may reach back into anything staged before it).
//   MODE 0: count symbol frequencies into cd, return the fixed-Huffman bits;
//   MODE 1: return the bits under cd's code tables;
//   MODE 2: write the codes at `pos` with cd's tables.
template <int MODE>
__device__ uint32_t parse_range(const uint8_t* buf, int base, int q0, int q1, const int* cand,
                                int ncand, Codes* cd, uint32_t* words, uint32_t pos) {
  uint32_t nbits = 0;
  int q = q0;
  while (q < q1) {
    const int at = base + q;
    const int maxl = min(258, q1 - q);
    int bl = 0, bd = 0;
    if (maxl >= 3) {
      const uint8_t x0 = buf[at], x1 = buf[at + 1], x2 = buf[at + 2];
      for (int c = 0; c < ncand; ++c) {
        const int d = cand[c];
        if (d > at) break;
        const uint8_t* a = buf + at;
        const uint8_t* b = a - d;
        if (b[0] != x0) continue;           // most candidates fail on the first byte
        if (b[1] != x1 || b[2] != x2) continue;
        int l = 3;
        while (l < maxl && a[l] == b[l]) ++l;
        if (l > bl) {
          bl = l;
          bd = d;
          if (l == maxl) break;
        }
      }
    }
    if (bl >= 3) {
      int sym, nx, xv, dsy, dnx, dxv;
      length_sym(bl, &sym, &nx, &xv);
      dist_sym(bd, &dsy, &dnx, &dxv);
      if (MODE == 0) {
        hist_add(cd->lf, sym);
        hist_add(cd->df, dsy);
        nbits += fixed_litlen_len(sym) + nx + 5 + dnx;
      } else {
        const int n1 = cd->llen[sym], n2 = cd->dlen[dsy];
        nbits += n1 + nx + n2 + dnx;
        if (MODE == 2) {
          put_bits(words, pos, cd->lcode[sym] | ((uint32_t)xv << n1), n1 + nx);
          put_bits(words, pos, cd->dcode[dsy] | ((uint32_t)dxv << n2), n2 + dnx);
        }
      }
      q += bl;
    } else {
      const int lit = buf[at];
      if (MODE == 0) {
        hist_add(cd->lf, lit);
        nbits += fixed_litlen_len(lit);
      } else {
        nbits += cd->llen[lit];
        if (MODE == 2) put_bits(words, pos, cd->lcode[lit], cd->llen[lit]);
      }
      q += 1;
    }
  }
  return nbits;
}

// Length-limited Huffman code lengths for n symbols with frequencies f (0 =
// unused): symbols ranked by (frequency, index) in parallel, then one thread
// runs the in-place minimum-redundancy construction of Moffat & Katajainen and
// clamps the lengths to maxlen, restoring the Kraft sum by moving leaves down
// from the deepest level that has room (longest codes to the rarest symbols).
__device__ void huff_lengths(const uint32_t* f, int n, int maxlen, uint8_t* len, Codes* cd) {
  __shared__ int m_sh;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    len[i] = 0;
    if (f[i] == 0) continue;
    int r = 0;
    for (int j = 0; j < n; ++j) r += f[j] != 0 && (f[j] < f[i] || (f[j] == f[i] && j < i));
    cd->sym[r] = (uint16_t)i;
    cd->A[r] = f[i];
  }
  if (threadIdx.x == 0) {
    int m = 0;
    for (int i = 0; i < n; ++i) m += f[i] != 0;
    m_sh = m;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int m = m_sh;
    uint32_t* A = cd->A;
    if (m == 1) {
      len[cd->sym[0]] = 1;
    } else if (m > 1) {
      // Moffat-Katajainen: A sorted ascending -> code lengths in place
      A[0] += A[1];
      int root = 0, leaf = 2;
      for (int next = 1; next < m - 1; ++next) {
        if (leaf >= m || A[root] < A[leaf]) { A[next] = A[root]; A[root++] = next; }
        else A[next] = A[leaf++];
        if (leaf >= m || (root < next && A[root] < A[leaf])) { A[next] += A[root]; A[root++] = next; }
        else A[next] += A[leaf++];
      }
      A[m - 2] = 0;
      for (int next = m - 3; next >= 0; --next) A[next] = A[A[next]] + 1;
      int avbl = 1, used = 0, dpth = 0, rt = m - 2, nx = m - 1;
      while (avbl > 0) {
        while (rt >= 0 && (int)A[rt] == dpth) { ++used; --rt; }
        while (avbl > used) { A[nx--] = dpth; --avbl; }
        avbl = 2 * used;
        ++dpth;
        used = 0;
      }
      // clamp to maxlen
      int num[33];
      for (int l = 0; l <= 32; ++l) num[l] = 0;
      for (int i = 0; i < m; ++i) num[min((int)A[i], 32)]++;
      for (int l = maxlen + 1; l <= 32; ++l) { num[maxlen] += num[l]; num[l] = 0; }
      uint32_t total = 0;
      for (int l = maxlen; l >= 1; --l) total += (uint32_t)num[l] << (maxlen - l);
      while (total != (1u << maxlen)) {
        num[maxlen]--;
        for (int l = maxlen - 1; l >= 1; --l)
          if (num[l]) { num[l]--; num[l + 1] += 2; break; }
        total--;
      }
      int i = 0;
      for (int l = maxlen; l >= 1; --l)
        for (int k = num[l]; k > 0; --k) len[cd->sym[i++]] = (uint8_t)l;
    }
  }
  __syncthreads();
}

// canonical codes from lengths (RFC 1951 3.2.2), bit-reversed
__device__ void canon_codes(const uint8_t* len, int n, uint16_t* code) {
  int cnt[16] = {0}, next[16];
  for (int i = 0; i < n; ++i) cnt[len[i]]++;
  cnt[0] = 0;
  int c = 0;
  for (int l = 1; l < 16; ++l) { c = (c + cnt[l - 1]) << 1; next[l] = c; }
  for (int i = 0; i < n; ++i)
    code[i] = len[i] ? (uint16_t)rev_bits((uint32_t)next[len[i]]++, len[i]) : 0;
}

// Dynamic-Huffman tables of the unit from cd->lf / cd->df, the run-length coded
// code lengths and the size of the block header (cd->header_bits).
__device__ void build_dynamic(Codes* cd) {
  if (threadIdx.x == 0) cd->lf[256] = 1;  // end of block
  __syncthreads();
  huff_lengths(cd->lf, 286, 15, cd->llen, cd);
  huff_lengths(cd->df, 30, 15, cd->dlen, cd);
  if (threadIdx.x == 0) {
    // a block without matches still declares one distance code of length 1
    bool any = false;
    for (int i = 0; i < 30; ++i) any |= cd->dlen[i] != 0;
    if (!any) cd->dlen[0] = 1;
    canon_codes(cd->llen, 286, cd->lcode);
    canon_codes(cd->dlen, 30, cd->dcode);
    int hlit = 286, hdist = 30;
    while (hlit > 257 && cd->llen[hlit - 1] == 0) --hlit;
    while (hdist > 1 && cd->dlen[hdist - 1] == 0) --hdist;
    cd->hlit = hlit;
    cd->hdist = hdist;
    // run-length code the concatenated code lengths (symbols 0-15, 16, 17, 18)
    const int N = hlit + hdist;
    auto L = [&](int i) { return i < hlit ? cd->llen[i] : cd->dlen[i - hlit]; };
    int nr = 0;
    for (int i = 0; i < 19; ++i) cd->cf[i] = 0;
    auto emit = [&](int sym, int extra) { cd->rle[nr++] = (uint16_t)(sym | (extra << 5)); cd->cf[sym]++; };
    for (int i = 0; i < N;) {
      const int v = L(i);
      int run = 1;
      while (i + run < N && L(i + run) == v) ++run;
      i += run;
      if (v == 0) {
        while (run >= 3) {
          const int r = min(run, 138);
          if (r >= 11) emit(18, r - 11);
          else emit(17, r - 3);
          run -= r;
        }
        while (run-- > 0) emit(0, 0);
      } else {
        emit(v, 0);
        --run;
        while (run >= 3) {
          const int r = min(run, 6);
          emit(16, r - 3);
          run -= r;
        }
        while (run-- > 0) emit(v, 0);
      }
    }
    cd->nrle = nr;
  }
  __syncthreads();
  huff_lengths(cd->cf, 19, 7, cd->clen, cd);
  if (threadIdx.x == 0) {
    canon_codes(cd->clen, 19, cd->ccode);
    const uint8_t order[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};
    int hclen = 19;
    while (hclen > 4 && cd->clen[order[hclen - 1]] == 0) --hclen;
    cd->hclen = hclen;
    uint32_t bits = 3 + 5 + 5 + 4 + 3 * hclen;
    for (int i = 0; i < cd->nrle; ++i) {
      const int sym = cd->rle[i] & 31;
      bits += cd->clen[sym] + (sym == 16 ? 2 : sym == 17 ? 3 : sym == 18 ? 7 : 0);
    }
    cd->header_bits = bits;
  }
  __syncthreads();
}

// block header (BFINAL = 0, BTYPE = 10) at bit 0, one thread
__device__ void write_dynamic_header(const Codes* cd, uint32_t* words) {
  const uint8_t order[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};
  uint32_t pos = 0;
  put_bits(words, pos, 4u, 3);
  put_bits(words, pos, (uint32_t)(cd->hlit - 257), 5);
  put_bits(words, pos, (uint32_t)(cd->hdist - 1), 5);
  put_bits(words, pos, (uint32_t)(cd->hclen - 4), 4);
  for (int i = 0; i < cd->hclen; ++i) put_bits(words, pos, cd->clen[order[i]], 3);
  for (int i = 0; i < cd->nrle; ++i) {
    const int sym = cd->rle[i] & 31, ex = cd->rle[i] >> 5;
    const int nx = sym == 16 ? 2 : sym == 17 ? 3 : sym == 18 ? 7 : 0;
    put_bits(words, pos, cd->ccode[sym] | ((uint32_t)ex << cd->clen[sym]), cd->clen[sym] + nx);
  }
}

__device__ void fixed_tables(Codes* cd) {
  for (int s = threadIdx.x; s < 288; s += blockDim.x) {
    uint32_t c;
    cd->llen[s] = (uint8_t)litlen_code(s, &c);
    cd->lcode[s] = (uint16_t)c;
  }
  for (int s = threadIdx.x; s < 32; s += blockDim.x) {
    cd->dlen[s] = 5;
    cd->dcode[s] = (uint16_t)rev_bits(s, 5);
  }
  __syncthreads();
}

__device__ __forceinline__ uint64_t block_exclusive_scan(uint64_t v, uint64_t* total) {
  __shared__ uint64_t wsum[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint64_t incl = v;
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint64_t s = lane < nw ? wsum[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t t = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += t;
    }
    if (lane < nw) wsum[lane] = s;  // inclusive warp prefix
  }
  __syncthreads();
  const uint64_t before = warp > 0 ? wsum[warp - 1] : 0;
  *total = wsum[nw - 1];
  __syncthreads();
  return before + incl - v;
}

constexpr size_t kDeflateSmem = 16 + kHist + kUnit + 16 + (kSlot + 64) + sizeof(Codes) + 16;

// Each unit is coded as the smallest of: one dynamic-Huffman block, one
// fixed-Huffman block, one stored block.
__global__ void __launch_bounds__(kDThreads) deflate_kernel(DeflateParams p) {
  extern __shared__ __align__(16) uint8_t dsm[];
  const int u = blockIdx.x;
  const UnitGeom g = unit_geom(p.stream_len, p.last_len, p.nstreams, p.upc, u);
  // stage [start - hist, start + len) with aligned 16-byte loads
  const uint8_t* src = p.data + g.start - g.hist;
  const int mis = (int)(reinterpret_cast<uintptr_t>(src) & 15);
  const uint4* s16 = reinterpret_cast<const uint4*>(src - mis);
  const int nvec = (mis + g.hist + g.len + 15) >> 4;
  uint4* stage = reinterpret_cast<uint4*>(dsm);
  for (int i = threadIdx.x; i < nvec; i += blockDim.x) stage[i] = s16[i];
  const uint8_t* buf = dsm + mis;            // buf[0] = first history byte
  uint32_t* words = reinterpret_cast<uint32_t*>(dsm + 16 + kHist + kUnit + 16);
  constexpr int kWords = (kSlot + 64) / 4;
  Codes* cd = reinterpret_cast<Codes*>(dsm + 16 + kHist + kUnit + 16 + kSlot + 64);
  for (int i = threadIdx.x; i < kWords; i += blockDim.x) words[i] = 0u;
  for (int i = threadIdx.x; i < 288; i += blockDim.x) cd->lf[i] = 0u;
  for (int i = threadIdx.x; i < 32; i += blockDim.x) cd->df[i] = 0u;
  __shared__ int cand[kMaxCand];
  if (threadIdx.x < kMaxCand) cand[threadIdx.x] = p.cand[threadIdx.x];
  const int ncand = p.ncand;
  __syncthreads();

  const int q0 = min(g.len, (int)threadIdx.x * kSub), q1 = min(g.len, q0 + kSub);
  // Adler-32 parts of this unit
  uint64_t sa = 0, sb = 0;
  for (int q = q0; q < q1; ++q) {
    const uint32_t b = buf[g.hist + q];
    sa += b;
    sb += (uint64_t)(g.len - q) * b;
  }
  const uint32_t nb_fixed = parse_range<0>(buf, g.hist, q0, q1, cand, ncand, cd, nullptr, 0);
  uint64_t fixed_bits;
  block_exclusive_scan(nb_fixed, &fixed_bits);
  {
    uint64_t t_sa, t_sb;
    block_exclusive_scan(sa, &t_sa);
    block_exclusive_scan(sb, &t_sb);
    if (threadIdx.x == 0) {
      p.uadler[2 * u] = (uint32_t)(t_sa % kAdlerMod);
      p.uadler[2 * u + 1] = (uint32_t)(t_sb % kAdlerMod);
    }
  }
  build_dynamic(cd);
  const uint32_t nb_dyn = parse_range<1>(buf, g.hist, q0, q1, cand, ncand, cd, nullptr, 0);
  uint64_t dyn_bits;
  const uint64_t dyn_before = block_exclusive_scan(nb_dyn, &dyn_bits);
  // block + end of block + empty stored block header (sync flush), padded,
  // then LEN = 0000, NLEN = FFFF
  const uint64_t dyn_total = cd->header_bits + dyn_bits + cd->llen[256] + 3;
  const uint64_t fixed_total = 3 + fixed_bits + 7 + 3;
  const bool use_dyn = dyn_total <= fixed_total;
  const uint64_t bits = use_dyn ? dyn_total : fixed_total;
  const int coded = (int)((bits + 7) >> 3) + 4;
  uint8_t* slot = p.slots + (size_t)u * kSlot;
  if (coded <= g.len + 5) {
    uint32_t pos;
    if (use_dyn) {
      if (threadIdx.x == 0) write_dynamic_header(cd, words);
      pos = cd->header_bits + (uint32_t)dyn_before;
    } else {
      // fixed path: recount positions under the fixed tables
      __syncthreads();
      fixed_tables(cd);
      const uint32_t nb = parse_range<1>(buf, g.hist, q0, q1, cand, ncand, cd, nullptr, 0);
      uint64_t tot;
      pos = 3 + (uint32_t)block_exclusive_scan(nb, &tot);
      if (threadIdx.x == 0) words[0] |= 2u;  // BFINAL = 0, BTYPE = 01
    }
    __syncthreads();
    parse_range<2>(buf, g.hist, q0, q1, cand, ncand, cd, words, pos);
    __syncthreads();
    if (threadIdx.x == 0) {  // end of block (zero bits for the fixed code)
      uint32_t e = (use_dyn ? cd->header_bits + (uint32_t)dyn_bits : 3 + (uint32_t)fixed_bits);
      put_bits(words, e, cd->lcode[256], cd->llen[256]);
    }
    __syncthreads();
    const uint8_t* wb = reinterpret_cast<const uint8_t*>(words);
    const int body = coded - 4;
    for (int i = threadIdx.x; i < coded; i += blockDim.x)
      slot[i] = i < body ? wb[i] : (i < body + 2 ? 0x00 : 0xFF);
    if (threadIdx.x == 0) p.ulen[u] = coded;
  } else {  // stored block: 00, LEN, NLEN, raw bytes
    for (int i = threadIdx.x; i < g.len + 5; i += blockDim.x) {
      uint8_t v;
      if (i == 0) v = 0x00;
      else if (i == 1) v = (uint8_t)(g.len & 0xFF);
      else if (i == 2) v = (uint8_t)(g.len >> 8);
      else if (i == 3) v = (uint8_t)(~g.len & 0xFF);
      else if (i == 4) v = (uint8_t)((~g.len >> 8) & 0xFF);
      else v = buf[g.hist + i - 5];
      slot[i] = v;
    }
    if (threadIdx.x == 0) p.ulen[u] = g.len + 5;
  }
}

struct FrameParams {
  int32_t mode;          // 0 = PNG (one stream, one IDAT chunk per unit), 1 = TIFF strips
  int32_t nstreams, upc, nunits;
  int64_t stream_len, last_len;
  const int32_t* ulen;
  const uint32_t* uadler;
  int64_t* udst;         // [nunits] where each unit's bytes go in `out`
  uint8_t* out;
  int64_t* out_len;
  int64_t* strip_bytes;  // TIFF: [nstreams]
};

__device__ __forceinline__ void put_be32(uint8_t* p, uint32_t v) {
  p[0] = (uint8_t)(v >> 24); p[1] = (uint8_t)(v >> 16); p[2] = (uint8_t)(v >> 8); p[3] = (uint8_t)v;
}

// Single CTA: unit offsets, stream framing, Adler-32 per stream.
__global__ void __launch_bounds__(1024) deflate_frame_kernel(FrameParams f) {
  __shared__ uint32_t crc_tab[256];
  crc_table(crc_tab);
  const int n = f.nunits;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int u0 = min(n, (int)threadIdx.x * per), u1 = min(n, u0 + per);
  uint64_t mine = 0;
  for (int u = u0; u < u1; ++u) mine += (uint64_t)f.ulen[u];
  uint64_t total;
  uint64_t pre = block_exclusive_scan(mine, &total);
  for (int u = u0; u < u1; ++u) {
    const int s = u / f.upc;
    // PNG: chunk u starts at P_u + 12 u + 2 (u > 0); data after len, type (+ 78 01 in chunk 0)
    // TIFF: strip s starts at P_(s upc) + 8 s; data after 78 01
    f.udst[u] = f.mode == 0 ? (int64_t)pre + 12 * (int64_t)u + 10 : (int64_t)pre + 8 * (int64_t)s + 2;
    pre += (uint64_t)f.ulen[u];
  }
  __syncthreads();
  // Adler-32 and framing per stream
  for (int s = threadIdx.x; s < f.nstreams; s += blockDim.x) {
    const int a0 = s * f.upc, a1 = min(n, a0 + f.upc);
    const int64_t slen = s == f.nstreams - 1 ? f.last_len : f.stream_len;
    uint64_t A = 1, Bs = (uint64_t)(slen % kAdlerMod);
    for (int u = a0; u < a1; ++u) {
      const int64_t off = (int64_t)(u - a0) * kUnit;
      const int64_t len = slen - off < kUnit ? slen - off : kUnit;
      const uint64_t a = f.uadler[2 * u], b = f.uadler[2 * u + 1];
      A += a;
      Bs += b + (uint64_t)((slen - off - len) % kAdlerMod) * a;
      A %= kAdlerMod;
      Bs %= kAdlerMod;
    }
    const uint32_t adler = (uint32_t)((Bs << 16) | A);
    const int64_t end = f.udst[a1 - 1] + f.ulen[a1 - 1];
    if (f.mode == 0) {
      // zlib header inside chunk 0; final chunk: 03 00 + Adler-32
      f.out[f.udst[0] - 2] = 0x78;
      f.out[f.udst[0] - 1] = 0x01;
      uint8_t* c = f.out + end + 4;  // after the last unit's CRC
      put_be32(c, 6u);
      c[4] = 'I'; c[5] = 'D'; c[6] = 'A'; c[7] = 'T';
      c[8] = 0x03; c[9] = 0x00;
      put_be32(c + 10, adler);
      put_be32(c + 14, crc_bytes(crc_tab, 0u, c + 4, 10));
      *f.out_len = end + 4 + 18;
    } else {
      const int64_t start = f.udst[a0] - 2;
      f.out[start] = 0x78;
      f.out[start + 1] = 0x01;
      f.out[end] = 0x03;
      f.out[end + 1] = 0x00;
      put_be32(f.out + end + 2, adler);
      f.strip_bytes[s] = end + 6 - start;
      if (s == f.nstreams - 1) *f.out_len = end + 6;
    }
  }
}

// One CTA per unit: copy into place; PNG adds chunk length, type and CRC-32.
__global__ void __launch_bounds__(256) deflate_place_kernel(FrameParams f, const uint8_t* __restrict__ slots) {
  __shared__ uint32_t crc_tab[256];
  __shared__ uint32_t part[256];
  crc_table(crc_tab);
  const int u = blockIdx.x;
  const int len = f.ulen[u];
  const uint8_t* src = slots + (size_t)u * kSlot;
  uint8_t* dst = f.out + f.udst[u];
  for (int i = threadIdx.x; i < len; i += blockDim.x) dst[i] = src[i];
  if (f.mode != 0) return;
  __syncthreads();
  // CRC of the data: pieces right-aligned so every right subtree of the merge
  // tree spans P 2^k bytes
  const int P = (len + blockDim.x - 1) / blockDim.x;
  const int t = threadIdx.x;
  const int e = len - ((int)blockDim.x - 1 - t) * P;
  const int b = max(0, e - P);
  part[t] = e > 0 ? crc_bytes(crc_tab, 0u, src + b, e - b) : 0u;
  uint32_t shift = x8nmodp((uint64_t)P);
  __syncthreads();
  for (int span = 1; span < (int)blockDim.x; span <<= 1) {
    if ((t & (2 * span - 1)) == 0) part[t] = multmodp(shift, part[t]) ^ part[t + span];
    shift = multmodp(shift, shift);
    __syncthreads();
  }
  if (t == 0) {
    uint8_t head[6] = {'I', 'D', 'A', 'T', 0x78, 0x01};
    const int hn = u == 0 ? 6 : 4;
    const uint32_t pre = crc_bytes(crc_tab, 0u, head, hn);
    const uint32_t crc = multmodp(x8nmodp((uint64_t)len), pre) ^ part[0];
    uint8_t* c = dst - (hn + 4);
    put_be32(c, (uint32_t)(len + hn - 4));
    c[4] = 'I'; c[5] = 'D'; c[6] = 'A'; c[7] = 'T';
    put_be32(dst + len, crc);
  }
}

// ------------------------------------------------------------------- host
cudaError_t init_crc_consts() {
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [&] {
    auto mul = [](uint32_t a, uint32_t b) {
      uint32_t m = 1u << 31, p = 0;
      for (;;) {
        if (a & m) {
          p ^= b;
          if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = (b & 1) ? (b >> 1) ^ kCrcPoly : b >> 1;
      }
      return p;
    };
    uint32_t t[32];
    t[0] = 1u << 30;  // x^1
    for (int k = 1; k < 32; ++k) t[k] = mul(t[k - 1], t[k - 1]);
    err = cudaMemcpyToSymbol(c_x2n, t, sizeof(t));
  });
  return err;
}

struct Plan {
  int64_t rb;          // raw bytes per image row
  int64_t filt_row;    // filtered bytes per row
  int64_t nstreams, stream_len, last_len, upc, nunits;
};

Plan make_plan(int64_t rows, int64_t cols, int channels, int depth, int format, int64_t rps) {
  Plan p{};
  p.rb = cols * channels * (depth / 8);
  if (format == 0) {
    p.filt_row = p.rb + 1;
    p.nstreams = 1;
    p.stream_len = rows * p.filt_row;
    p.last_len = p.stream_len;
  } else {
    p.filt_row = p.rb;
    p.nstreams = (rows + rps - 1) / rps;
    p.stream_len = rps * p.rb;
    p.last_len = (rows - (p.nstreams - 1) * rps) * p.rb;
  }
  p.upc = (p.stream_len + kUnit - 1) / kUnit;
  const int64_t last_units = (p.last_len + kUnit - 1) / kUnit;
  p.nunits = (p.nstreams - 1) * p.upc + last_units;
  return p;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct Ws {
  uint8_t* filt;
  uint8_t* slots;
  int32_t* ulen;
  uint32_t* uadler;
  int64_t* udst;
};
size_t ws_layout(const Plan& p, Ws* w, void* base) {
  size_t off = 0;
  const size_t o_filt = off; off += align256((size_t)(p.stream_len * (p.nstreams - 1) + p.last_len) + 16);
  const size_t o_slots = off; off += align256((size_t)p.nunits * kSlot);
  const size_t o_ulen = off; off += align256((size_t)p.nunits * 4);
  const size_t o_adl = off; off += align256((size_t)p.nunits * 8);
  const size_t o_dst = off; off += align256((size_t)p.nunits * 8);
  if (w && base) {
    char* b = static_cast<char*>(base);
    w->filt = reinterpret_cast<uint8_t*>(b + o_filt);
    w->slots = reinterpret_cast<uint8_t*>(b + o_slots);
    w->ulen = reinterpret_cast<int32_t*>(b + o_ulen);
    w->uadler = reinterpret_cast<uint32_t*>(b + o_adl);
    w->udst = reinterpret_cast<int64_t*>(b + o_dst);
  }
  return off;
}

int64_t out_bound(const Plan& p, int format) {
  // every unit at most its stored form; PNG: 12 bytes of chunk per unit + zlib
  // header + the final chunk; TIFF: 8 bytes of zlib framing per strip
  const int64_t raw = p.stream_len * (p.nstreams - 1) + p.last_len;
  return raw + 5 * p.nunits + (format == 0 ? 12 * p.nunits + 2 + 18 : 8 * p.nstreams) + 64;
}

int check_image(int64_t rows, int64_t cols, int channels, int depth) {
  UT_REQUIRE(rows > 0 && cols > 0, "image must be non-empty, got %lldx%lld", (long long)rows,
             (long long)cols);
  UT_REQUIRE(channels == 1 || channels == 3, "image must have 1 or 3 channels, got %d", channels);
  UT_REQUIRE(depth == 8 || depth == 16, "image depth must be 8 or 16, got %d", depth);
  UT_REQUIRE(rows < (1LL << 31) && cols < (1LL << 31), "image too large");
  return UT_OK;
}

int fill_cands(DeflateParams& dp, int64_t stride, int bpp) {
  const int64_t want[] = {1, 2, 3, 4, bpp, 2 * (int64_t)bpp, stride - bpp, stride, stride + bpp,
                          2 * stride};
  int64_t c[kMaxCand];
  int n = 0;
  for (int64_t d : want) {
    if (d < 1 || d > 32768) continue;
    bool dup = false;
    for (int i = 0; i < n; ++i) dup |= c[i] == d;
    if (!dup && n < kMaxCand) c[n++] = d;
  }
  for (int i = 1; i < n; ++i)  // ascending
    for (int j = i; j > 0 && c[j - 1] > c[j]; --j) { const int64_t t = c[j]; c[j] = c[j - 1]; c[j - 1] = t; }
  dp.ncand = n;
  for (int i = 0; i < n; ++i) dp.cand[i] = (int32_t)c[i];
  return n;
}

int run_deflate(const Plan& pl, const Ws& w, int format, int bpp, uint8_t* out, int64_t* out_len,
                int64_t* strip_bytes, cudaStream_t st) {
  if (cudaError_t e = init_crc_consts()) return cuda_status(e, "CRC constants");
  DeflateParams dp{};
  dp.data = w.filt;
  dp.stream_len = pl.stream_len;
  dp.last_len = pl.last_len;
  dp.nstreams = (int32_t)pl.nstreams;
  dp.upc = (int32_t)pl.upc;
  dp.nunits = (int32_t)pl.nunits;
  fill_cands(dp, pl.filt_row, bpp);
  dp.slots = w.slots;
  dp.ulen = w.ulen;
  dp.uadler = w.uadler;
  static SmemAttr attr;
  if (int rc = ensure_smem(attr, deflate_kernel, kDeflateSmem, "deflate smem attribute")) return rc;
  deflate_kernel<<<(unsigned)pl.nunits, kDThreads, kDeflateSmem, st>>>(dp);
  UT_CHECK_LAUNCH("deflate_kernel");
  FrameParams fp{};
  fp.mode = format == 0 ? 0 : 1;
  fp.nstreams = dp.nstreams;
  fp.upc = dp.upc;
  fp.nunits = dp.nunits;
  fp.stream_len = pl.stream_len;
  fp.last_len = pl.last_len;
  fp.ulen = w.ulen;
  fp.uadler = w.uadler;
  fp.udst = w.udst;
  fp.out = out;
  fp.out_len = out_len;
  fp.strip_bytes = strip_bytes;
  deflate_frame_kernel<<<1, 1024, 0, st>>>(fp);
  UT_CHECK_LAUNCH("deflate_frame_kernel");
  deflate_place_kernel<<<(unsigned)pl.nunits, 256, 0, st>>>(fp, w.slots);
  UT_CHECK_LAUNCH("deflate_place_kernel");
  return UT_OK;
}

}  // namespace
}  // namespace ut

using namespace ut;

extern "C" {

size_t ut_encode_ws(int64_t rows, int64_t cols, int32_t channels, int32_t depth, int32_t format,
                    int64_t rows_per_strip) {
  if (rows <= 0 || cols <= 0 || (format != 0 && rows_per_strip <= 0)) return 0;
  return ws_layout(make_plan(rows, cols, channels, depth, format, rows_per_strip), nullptr, nullptr);
}

int64_t ut_encode_bound(int64_t rows, int64_t cols, int32_t channels, int32_t depth, int32_t format,
                        int64_t rows_per_strip) {
  if (rows <= 0 || cols <= 0 || (format != 0 && rows_per_strip <= 0)) return 0;
  return out_bound(make_plan(rows, cols, channels, depth, format, rows_per_strip), format);
}

int ut_encode_png(const void* img, int64_t rows, int64_t cols, int32_t channels, int32_t depth,
                  uint8_t* out, int64_t out_cap, int64_t* out_len, void* ws, size_t ws_bytes,
                  void* stream) {
  if (int rc = check_image(rows, cols, channels, depth)) return rc;
  UT_REQUIRE(img && out && out_len && ws, "ut_encode_png: null pointer");
  const Plan pl = make_plan(rows, cols, channels, depth, 0, 1);
  Ws w;
  const size_t need = ws_layout(pl, &w, ws);
  UT_REQUIRE(ws_bytes >= need, "ut_encode_png: workspace %zu < %zu", ws_bytes, need);
  UT_REQUIRE(out_cap >= out_bound(pl, 0), "ut_encode_png: output capacity %lld < %lld",
             (long long)out_cap, (long long)out_bound(pl, 0));
  cudaStream_t st = as_stream(stream);
  const int bpp = channels * (depth / 8);
  png_filter_kernel<<<(unsigned)rows, 256, 0, st>>>(static_cast<const uint8_t*>(img), pl.rb, depth,
                                                    bpp, w.filt);
  UT_CHECK_LAUNCH("png_filter_kernel");
  return run_deflate(pl, w, 0, bpp, out, out_len, nullptr, st);
}

int ut_encode_tiff(const void* img, int64_t rows, int64_t cols, int32_t channels, int32_t depth,
                   int32_t compression, int64_t rows_per_strip, uint8_t* out, int64_t out_cap,
                   int64_t* strip_bytes, int64_t* out_len, void* ws, size_t ws_bytes, void* stream) {
  if (int rc = check_image(rows, cols, channels, depth)) return rc;
  UT_REQUIRE(compression == 1 || compression == 8, "TIFF compression must be 1 (none) or 8 (deflate), got %d",
             compression);
  UT_REQUIRE(rows_per_strip > 0, "rows_per_strip must be positive");
  UT_REQUIRE(img && out && out_len && strip_bytes, "ut_encode_tiff: null pointer");
  const Plan pl = make_plan(rows, cols, channels, depth, 1, rows_per_strip);
  cudaStream_t st = as_stream(stream);
  const int64_t raw = pl.rb * rows;
  if (compression == 1) {
    UT_REQUIRE(out_cap >= raw, "ut_encode_tiff: output capacity %lld < %lld", (long long)out_cap,
               (long long)raw);
    cudaError_t e = cudaMemcpyAsync(out, img, (size_t)raw, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_status(e, "ut_encode_tiff copy");
    std::vector<int64_t> sb((size_t)pl.nstreams, pl.stream_len);
    sb.back() = pl.last_len;
    int64_t total = raw;
    e = cudaMemcpyAsync(strip_bytes, sb.data(), sb.size() * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out_len, &total, 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // host staging buffers above
    if (e != cudaSuccess) return cuda_status(e, "ut_encode_tiff sizes");
    return UT_OK;
  }
  UT_REQUIRE(ws, "ut_encode_tiff: null workspace");
  Ws w;
  const size_t need = ws_layout(pl, &w, ws);
  UT_REQUIRE(ws_bytes >= need, "ut_encode_tiff: workspace %zu < %zu", ws_bytes, need);
  UT_REQUIRE(out_cap >= out_bound(pl, 1), "ut_encode_tiff: output capacity %lld < %lld",
             (long long)out_cap, (long long)out_bound(pl, 1));
  const int64_t spr = cols * channels;
  const int64_t n = rows * spr;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
  if (depth == 8)
    tiff_predict_kernel<uint8_t><<<grid, 256, 0, st>>>(static_cast<const uint8_t*>(img), rows, spr,
                                                       channels, w.filt);
  else
    tiff_predict_kernel<uint16_t><<<grid, 256, 0, st>>>(static_cast<const uint16_t*>(img), rows, spr,
                                                        channels, reinterpret_cast<uint16_t*>(w.filt));
  UT_CHECK_LAUNCH("tiff_predict_kernel");
  return run_deflate(pl, w, 1, channels * (depth / 8), out, out_len, strip_bytes, st);
}

}  // extern "C"
