// kvf_band.cu — shared-memory staged tile transposes for tilings whose tile
// rows are narrower than 8 channels (b_d in {1, 2, 4}), sm_100a.
//
// In those layouts (fk/layout.py:94-106, e.g. (a_h, b_h, a_d, b_d) = (1, 8,
// 128, 1) or (2, 4, 32, 4)) consecutive channels of a head sit b_d bytes apart
// in a column of tile rows (fk/layout.py:244-250: h = i_h*b_h + j_h,
// d = i_d*b_d + j_d -> row i_h*a_d + i_d, column j_h*b_d + j_d), so a thread
// reading 8 consecutive channels from global memory would touch 8 / b_d rows.
// Instead a CTA owns whole BANDS = one grid row of tiles of one frame plane
// (tile_h pixel rows x frame_w bytes, contiguous rows at the surface pitch):
//
//   restore: band rows -> shared memory with 16-B coalesced loads; each lane
//            then gathers one output block = NHB = 4 / b_d heads x 8 channels
//            as 8 / b_d 32-bit words (column j_h0*b_d, rows i_h*a_d + d0/b_d
//            + r), transposes them in registers (byte permutes) into NHB
//            8-sample vectors, dequantises and writes NHB 16-B slot stores
//            (fk/fetchsim.py:347-355 + fk/kvmodel.py:147-152);
//   pack:    the reverse: 16-B source loads, exact quantisation
//            (fk/kvmodel.py:141-143), the transpose into words, shared-memory
//            writes, then the band leaves with 16-B coalesced stores; pad
//            tiles stay 128 (fk/layout.py:231, 251-253).
//
// Shared-memory words are XOR-swizzled by row (word ^ (row >> log2(8/b_d)) ^
// (row mod 8/b_d)) so the 32 lanes of a warp, whose blocks are 8/b_d rows
// apart, hit different banks, and so do consecutive rows of the band fill.  Requires tile_w = b_h*b_d >= 4 (a 32-bit word holds NHB
// heads of one tile row); narrower tiles use the one-thread-per-sample kernels.
#include <algorithm>
#include <vector>

#include "kvf_pack_common.cuh"

namespace kvf {

namespace {

constexpr int kBThreads = 256;
constexpr int kBWarps = kBThreads / 32;
// per CTA: the default 48 KB limit covers static + dynamic shared memory, so
// the bands stay below it with room for the kernels' static arrays
constexpr int kBandSmem = 46 * 1024;

// Band geometry of a unit (host-derived).
struct BandGeom {
  int32_t tile_h, tile_w, grid_cols, grid_rows;
  int32_t frame_w;
  int32_t lg_sp;        // shared row pitch = 2^lg_sp bytes >= frame_w (>= 16)
  int32_t band_bytes;   // tile_h << lg_sp
  int32_t nb;           // bands per CTA
  int32_t g16;          // global band rows move as 16-B pieces (else 4-B)
  int32_t gpr;          // pieces per band row
  int32_t lg_th;        // log2 tile_h
  FastDiv div_gpr, div_cols, div_rows;
};

inline int lg2i(int64_t v) {
  int r = 0;
  while ((int64_t(1) << r) < v) ++r;
  return r;
}

inline BandGeom make_band(const kvf_plan& p, const kvf_surface& fr) {
  BandGeom b;
  b.tile_h = p.a_h * p.a_d;
  b.tile_w = p.b_h * p.b_d;
  b.grid_cols = p.grid_cols;
  b.grid_rows = p.grid_rows;
  b.frame_w = p.frame_w;
  b.lg_sp = std::max(4, lg2i(p.frame_w));
  b.band_bytes = b.tile_h << b.lg_sp;
  const int want = (16 + b.grid_cols - 1) / b.grid_cols;  // >= 16 tiles per CTA
  b.nb = std::max(1, std::min(std::min(want, 16), kBandSmem / std::max(1, b.band_bytes)));
  b.g16 = (p.frame_w % 16 == 0 && fr.row_pitch % 16 == 0 && fr.plane_stride % 16 == 0 &&
           fr.frame_stride % 16 == 0 && reinterpret_cast<uintptr_t>(fr.base) % 16 == 0);
  b.gpr = b.g16 ? p.frame_w / 16 : p.frame_w / 4;
  b.lg_th = lg2i(b.tile_h);
  b.div_gpr = make_fastdiv(b.gpr);
  b.div_cols = make_fastdiv(p.grid_cols);
  b.div_rows = make_fastdiv(p.grid_rows);
  return b;
}

// Shared byte offset of 32-bit word `w` of row `r` of a band (swizzled).
template <int BD>
__device__ __forceinline__ uint32_t band_word(const BandGeom& b, int r, int w) {
  constexpr int LGR = BD == 1 ? 3 : (BD == 2 ? 2 : 1);  // rows per lane block: 8 / BD
  const int mask = (1 << (b.lg_sp - 2)) - 1;
  // rows of one lane block share the high part (lanes differ in it); the low
  // part spreads consecutive rows (band fill) over banks
  const int sw = (r >> LGR) ^ (r & ((1 << LGR) - 1));
  return ((uint32_t)r << b.lg_sp) + (uint32_t)((w ^ sw) & mask) * 4u;
}

// NHB = 4/BD heads x 8 channels <-> 8/BD words of a tile column.  Word r holds,
// at byte j*BD + e, head j's channel r*BD + e.
template <int BD>
__device__ __forceinline__ void words_to_vecs(const uint32_t (&w)[8 / BD], uint2 (&o)[4 / BD]) {
  if constexpr (BD == 4) {
    o[0] = make_uint2(w[0], w[1]);
  } else if constexpr (BD == 2) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint32_t sel = j == 0 ? 0x5410u : 0x7632u;
      o[j] = make_uint2(__byte_perm(w[0], w[1], sel), __byte_perm(w[2], w[3], sel));
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      // bytes j of w0..w3 -> one word, of w4..w7 -> the other
      const uint32_t lo01 = __byte_perm(w[0], w[1], (uint32_t)(j | ((j + 4) << 4)));
      const uint32_t lo23 = __byte_perm(w[2], w[3], (uint32_t)(j | ((j + 4) << 4)));
      const uint32_t hi01 = __byte_perm(w[4], w[5], (uint32_t)(j | ((j + 4) << 4)));
      const uint32_t hi23 = __byte_perm(w[6], w[7], (uint32_t)(j | ((j + 4) << 4)));
      o[j] = make_uint2(__byte_perm(lo01, lo23, 0x5410u), __byte_perm(hi01, hi23, 0x5410u));
    }
  }
}

template <int BD>
__device__ __forceinline__ void vecs_to_words(const uint2 (&o)[4 / BD], uint32_t (&w)[8 / BD]) {
  if constexpr (BD == 4) {
    w[0] = o[0].x;
    w[1] = o[0].y;
  } else if constexpr (BD == 2) {
    // head 0 channels (a0 a1 | a2 a3 | ...), head 1 (b0 b1 | ...): word r = a(2r) a(2r+1) b(2r) b(2r+1)
    w[0] = __byte_perm(o[0].x, o[1].x, 0x5410u);
    w[1] = __byte_perm(o[0].x, o[1].x, 0x7632u);
    w[2] = __byte_perm(o[0].y, o[1].y, 0x5410u);
    w[3] = __byte_perm(o[0].y, o[1].y, 0x7632u);
  } else {
    // word r = channel r of heads 0..3
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int sh = r & 3;
      const uint32_t a = r < 4 ? o[0].x : o[0].y, b = r < 4 ? o[1].x : o[1].y;
      const uint32_t c = r < 4 ? o[2].x : o[2].y, d = r < 4 ? o[3].x : o[3].y;
      const uint32_t ab = __byte_perm(a, b, (uint32_t)(sh | ((sh + 4) << 4)));
      const uint32_t cd = __byte_perm(c, d, (uint32_t)(sh | ((sh + 4) << 4)));
      w[r] = __byte_perm(ab, cd, 0x5410u);
    }
  }
}

// Lane block -> (first head h0, first channel d0, tile row of word 0, word column).
struct Block {
  int h0, d0, row0, wcol;
};
__device__ __forceinline__ Block lane_block(const Geom& g, int blk, int nhb, int tc, int tile_w) {
  const int lg_dv = g.lg_D - 3;  // 8-channel blocks per head: D / 8
  Block k;
  k.d0 = (blk & ((1 << lg_dv) - 1)) << 3;
  k.h0 = (blk >> lg_dv) * nhb;
  const int i_h = k.h0 >> g.lg_bh, j_h0 = k.h0 & ((1 << g.lg_bh) - 1);
  k.row0 = i_h * g.a_d + (k.d0 >> g.lg_bd);
  k.wcol = (tc * tile_w + (j_h0 << g.lg_bd)) >> 2;
  return k;
}

// ------------------------------------------------------------------ restore
struct RBandUnit {
  kvf_surface fr;
  Geom g;
  BandGeom b;
  const float* scales;
  kvf_paged dst;
  FastDiv div_bs;
  int32_t first_frame, n_bands, G;
};
struct RBandParams {
  int32_t n_units;
  RBandUnit u[KVF_MAX_UNITS / 2];
};
static_assert(sizeof(RBandParams) <= 32000, "kernel parameters above 32 KB");

template <int OUT, int BD>
__global__ void __launch_bounds__(kBThreads)
    restore_band_kernel(const __grid_constant__ RBandParams P) {
  extern __shared__ __align__(16) uint8_t s_band[];
  constexpr int NHB = 4 / BD, NW = 8 / BD;
  constexpr int ES = OUT == KVF_F32 ? 4 : (OUT == KVF_I8 ? 1 : 2);
  const RBandUnit& U = P.u[blockIdx.y];
  const int p = blockIdx.z;
  const BandGeom& B = U.b;
  const int j0 = blockIdx.x * B.nb;
  char* layer = reinterpret_cast<char*>(U.dst.layer[p]);
  if (j0 >= U.n_bands || layer == nullptr) return;
  const int nb = min(B.nb, U.n_bands - j0);
  const uint8_t* plane = U.fr.base + (int64_t)p * U.fr.plane_stride;
  // 1. bands -> shared (swizzled words); 4 pieces per thread in flight
  const int n_pieces = (nb * B.tile_h) * B.gpr;
  __shared__ const uint8_t* s_row0[16];  // first pixel row of each band (nb <= 16)
  if (threadIdx.x < nb) {
    const int j = j0 + threadIdx.x;
    const int fj = fdiv(B.div_rows, j);
    s_row0[threadIdx.x] = plane + (int64_t)(U.first_frame + fj) * U.fr.frame_stride +
                          (int64_t)(j - fj * B.grid_rows) * B.tile_h * U.fr.row_pitch;
  }
  __syncthreads();
  auto piece_src = [&](int x, int& r, uint8_t*& sb, int& piece) {
    const int row_all = fdiv(B.div_gpr, x);
    piece = x - row_all * B.gpr;
    const int b = row_all >> B.lg_th;
    r = row_all & (B.tile_h - 1);
    sb = s_band + b * B.band_bytes;
    return s_row0[b] + (int64_t)r * U.fr.row_pitch;
  };
  for (int x0 = threadIdx.x; x0 < n_pieces; x0 += 4 * kBThreads) {
    if (B.g16) {
      uint4 v[4];
      int rr[4], pc[4];
      uint8_t* sbs[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int x = x0 + u * kBThreads;
        if (x < n_pieces) v[u] = ld_nc_v4(piece_src(x, rr[u], sbs[u], pc[u]) + pc[u] * 16);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (x0 + u * kBThreads >= n_pieces) break;
        const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          *reinterpret_cast<uint32_t*>(sbs[u] + band_word<BD>(B, rr[u], pc[u] * 4 + e)) = w[e];
      }
    } else {
      for (int u = 0; u < 4; ++u) {
        const int x = x0 + u * kBThreads;
        if (x >= n_pieces) break;
        int r, pc;
        uint8_t* sb;
        const uint8_t* src = piece_src(x, r, sb, pc);
        *reinterpret_cast<uint32_t*>(sb + band_word<BD>(B, r, pc)) =
            __ldg(reinterpret_cast<const uint32_t*>(src + pc * 4));
      }
    }
  }
  __syncthreads();
  // 2. tiles -> slots.  Per lane: its blocks' tile rows, word columns, slot
  // offsets and group scales, computed once per CTA (independent of the tile).
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nblk = U.g.C / (8 * NHB);
  constexpr int MAXQ = 4 / NHB;  // blocks per lane for C <= 1024 * NHB
  const int64_t hs_b = U.dst.head_stride * ES;
  // one block: NW words of rows row0.., column wcol -> NHB 8-sample slot vectors
  auto do_block = [&](const uint8_t* sb, int row0, int wcol, char* dst0, const float* sc) {
    uint32_t w[NW];
#pragma unroll
    for (int r = 0; r < NW; ++r)
      w[r] = *reinterpret_cast<const uint32_t*>(sb + band_word<BD>(B, row0 + r, wcol));
#pragma unroll
    for (int jh = 0; jh < NHB; ++jh) {
      char* dst = dst0 + jh * hs_b;
      if constexpr (OUT == KVF_I8) {
        uint2 v[NHB];
        words_to_vecs<BD>(w, v);
        st_v2(dst, make_uint2(v[jh].x ^ 0x80808080u, v[jh].y ^ 0x80808080u));
      } else {
        // sample n of head jh is byte jh*BD + n%BD of word n/BD: straight to
        // the float 2^23 + sample (byte permute), then packed (q - 128) * s
        const uint64_t off2 = 0x4B0000804B000080ull, s2 = f2_pack(sc[jh], sc[jh]);
        float q[8];
#pragma unroll
        for (int n = 0; n < 8; n += 2) {
          const uint32_t lo = __byte_perm(w[n / BD], 0x4B000000u,
                                          0x7440u | (uint32_t)(jh * BD + n % BD));
          const uint32_t hi = __byte_perm(w[(n + 1) / BD], 0x4B000000u,
                                          0x7440u | (uint32_t)(jh * BD + (n + 1) % BD));
          const uint64_t y =
              f2_mul(f2_sub(f2_pack(__uint_as_float(lo), __uint_as_float(hi)), off2), s2);
          f2_unpack(y, q[n], q[n + 1]);
        }
        if constexpr (OUT == KVF_F32) {
          st_v4(dst, make_uint4(__float_as_uint(q[0]), __float_as_uint(q[1]),
                                __float_as_uint(q[2]), __float_as_uint(q[3])));
          st_v4(dst + 16, make_uint4(__float_as_uint(q[4]), __float_as_uint(q[5]),
                                     __float_as_uint(q[6]), __float_as_uint(q[7])));
        } else if constexpr (OUT == KVF_BF16) {
          st_v4(dst, make_uint4(pack_bf16x2(q[0], q[1]), pack_bf16x2(q[2], q[3]),
                                pack_bf16x2(q[4], q[5]), pack_bf16x2(q[6], q[7])));
        } else {
          st_v4(dst, make_uint4(pack_f16x2(q[0], q[1]), pack_f16x2(q[2], q[3]),
                                pack_f16x2(q[4], q[5]), pack_f16x2(q[6], q[7])));
        }
      }
    }
  };
  auto block_scales = [&](const Block& k, float* sc) {
#pragma unroll
    for (int jh = 0; jh < NHB; ++jh)
      sc[jh] = OUT == KVF_I8 ? 1.0f
                             : __ldg(U.scales + p * U.G +
                                     (((k.h0 + jh) * (1 << U.g.lg_D) + k.d0) >> U.g.lg_gs));
  };
  const bool pre = nblk <= 32 * MAXQ;
  int q_row0[MAXQ], q_wc[MAXQ];
  int64_t q_off[MAXQ];
  float q_sc[MAXQ][NHB];
  if (pre) {
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) {
      const int blk = lane + 32 * q;
      const Block k = lane_block(U.g, blk < nblk ? blk : 0, NHB, 0, B.tile_w);
      q_row0[q] = k.row0;
      q_wc[q] = blk < nblk ? k.wcol : -1;
      q_off[q] = ((int64_t)k.h0 * U.dst.head_stride + k.d0) * ES;
      block_scales(k, q_sc[q]);
    }
  }
  const int tw4 = B.tile_w >> 2;
  for (int t = warp; t < nb * B.grid_cols; t += kBWarps) {
    const int b = fdiv(B.div_cols, t), tc = t - b * B.grid_cols;
    const int j = j0 + b;
    const int fj = fdiv(B.div_rows, j);
    const int f = U.first_frame + fj, gr = j - fj * B.grid_rows;
    const int i = token_of(U.g, f, gr * B.grid_cols + tc);
    if (i >= U.g.T) continue;  // pad tile (uniform over the warp)
    char* slot = layer + paged_slot_offset_fd(U.dst, U.div_bs, i) * ES;
    const uint8_t* sb = s_band + b * B.band_bytes;
    if (pre) {
#pragma unroll
      for (int q = 0; q < MAXQ; ++q)
        if (q_wc[q] >= 0) do_block(sb, q_row0[q], tc * tw4 + q_wc[q], slot + q_off[q], q_sc[q]);
    } else {
      for (int blk = lane; blk < nblk; blk += 32) {
        const Block k = lane_block(U.g, blk, NHB, tc, B.tile_w);
        float sc[NHB];
        block_scales(k, sc);
        do_block(sb, k.row0, k.wcol, slot + ((int64_t)k.h0 * U.dst.head_stride + k.d0) * ES, sc);
      }
    }
  }
}

// --------------------------------------------------------------------- pack
struct PBandUnit {
  kvf_paged src;
  Geom g;
  BandGeom b;
  const float* scales;
  kvf_surface fr;
  FastDiv div_bs;
  int32_t n_bands, G;
};
struct PBandParams {
  int32_t n_units;
  PBandUnit u[kMaxPackUnits / 2];
};
static_assert(sizeof(PBandParams) <= 32000, "kernel parameters above 32 KB");
static_assert(kBandSmem / 16 >= 1, "");

template <int SRC, int BD>
__global__ void __launch_bounds__(kBThreads)
    pack_band_kernel(const __grid_constant__ PBandParams P) {
  extern __shared__ __align__(16) uint8_t s_band[];
  constexpr int NHB = 4 / BD, NW = 8 / BD;
  constexpr int ES = SRC == KVF_F32 ? 4 : (SRC == KVF_I8 ? 1 : 2);
  const PBandUnit& U = P.u[blockIdx.y];
  const int p = blockIdx.z;
  const BandGeom& B = U.b;
  const int j0 = blockIdx.x * B.nb;
  if (j0 >= U.n_bands) return;
  const int nb = min(B.nb, U.n_bands - j0);
  const char* layer = reinterpret_cast<const char*>(U.src.layer[p]);
  // 1. the CTA's bands start as pad bytes (128)
  {
    uint4* s4 = reinterpret_cast<uint4*>(s_band);
    const int n4 = (nb * B.band_bytes) >> 4;
    for (int x = threadIdx.x; x < n4; x += kBThreads)
      s4[x] = make_uint4(0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u);
  }
  __syncthreads();
  // 2. slots -> quantised tile words in shared memory
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nblk = U.g.C / (8 * NHB);
  if (layer != nullptr) {
    const int n_tiles = nb * B.grid_cols;
    constexpr int MAXQ = 4 / NHB;  // blocks per lane for C <= 1024 * NHB
    const int64_t hs_b = U.src.head_stride * ES;
    const int tw4 = B.tile_w >> 2;
    // one block of one tile: NHB source vectors -> quantised -> NW band words
    auto finish = [&](uint8_t* sb, int row0, int wcol, Raw8<SRC> (&raw)[NHB], const float* sc,
                      const float* inv) {
      uint2 v[NHB];
#pragma unroll
      for (int jh = 0; jh < NHB; ++jh) {
        if constexpr (SRC == KVF_I8) {
          v[jh] = make_uint2(raw[jh].a.x ^ 0x80808080u, raw[jh].a.y ^ 0x80808080u);
        } else {
          float x[8];
          raw8_to_float<SRC>(raw[jh], x);
          bool bad = false;  // scales may be caller-given: range checked too
          v[jh] = quantize8_fast<true>(x, inv[jh], bad);
          if (__builtin_expect(bad, 0))
            v[jh] = quantize8_exact(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7], sc[jh],
                                    inv[jh]);
        }
      }
      uint32_t w[NW];
      vecs_to_words<BD>(v, w);
#pragma unroll
      for (int r = 0; r < NW; ++r)
        *reinterpret_cast<uint32_t*>(sb + band_word<BD>(B, row0 + r, wcol)) = w[r];
    };
    auto load_block = [&](const char* src0, Raw8<SRC> (&raw)[NHB]) {
#pragma unroll
      for (int jh = 0; jh < NHB; ++jh) {
        if constexpr (SRC == KVF_I8) {
          const uint2 c = ld_nc_v2(src0 + jh * hs_b);  // 8 int8 codes
          raw[jh].a = make_uint4(c.x, c.y, 0u, 0u);
        } else {
          raw[jh] = load_raw8<SRC>(src0 + jh * hs_b);
        }
      }
    };
    auto block_scales = [&](const Block& k, float* sc, float* inv) {
#pragma unroll
      for (int jh = 0; jh < NHB; ++jh) {
        sc[jh] = SRC == KVF_I8 ? 1.0f
                               : __ldg(U.scales + p * U.G +
                                       (((k.h0 + jh) * (1 << U.g.lg_D) + k.d0) >> U.g.lg_gs));
        inv[jh] = __frcp_rn(sc[jh]);
      }
    };
    auto tile_of = [&](int t, const char*& slot, uint8_t*& sb, int& tc) {
      slot = nullptr;
      sb = s_band;
      tc = 0;
      if (t >= n_tiles) return;
      const int b = fdiv(B.div_cols, t);
      tc = t - b * B.grid_cols;
      const int j = j0 + b;
      const int f = fdiv(B.div_rows, j), gr = j - f * B.grid_rows;
      const int i = token_of(U.g, f, gr * B.grid_cols + tc);
      sb = s_band + b * B.band_bytes;
      if (i < U.g.T) slot = layer + paged_slot_offset_fd(U.src, U.div_bs, i) * ES;
    };
    if (nblk <= 32 * MAXQ) {
      // per-lane blocks, computed once
      int q_row0[MAXQ], q_wc[MAXQ];
      int64_t q_off[MAXQ];
      float q_sc[MAXQ][NHB], q_inv[MAXQ][NHB];
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int blk = lane + 32 * q;
        const Block k = lane_block(U.g, blk < nblk ? blk : 0, NHB, 0, B.tile_w);
        q_row0[q] = k.row0;
        q_wc[q] = blk < nblk ? k.wcol : -1;
        q_off[q] = ((int64_t)k.h0 * U.src.head_stride + k.d0) * ES;
        block_scales(k, q_sc[q], q_inv[q]);
      }
      // TU tiles per warp iteration (their source loads issued together):
      // two when a lane holds one block per tile, else the blocks suffice
      constexpr int TU = MAXQ == 1 ? 2 : 1;
      for (int t0 = warp; t0 < n_tiles; t0 += TU * kBWarps) {
        const char* slot[TU];
        uint8_t* sb[TU];
        int tc[TU];
#pragma unroll
        for (int u = 0; u < TU; ++u) tile_of(t0 + u * kBWarps, slot[u], sb[u], tc[u]);
        Raw8<SRC> raw[TU][MAXQ][NHB];
#pragma unroll
        for (int u = 0; u < TU; ++u)
#pragma unroll
          for (int q = 0; q < MAXQ; ++q)
            if (slot[u] != nullptr && q_wc[q] >= 0) load_block(slot[u] + q_off[q], raw[u][q]);
#pragma unroll
        for (int u = 0; u < TU; ++u)
#pragma unroll
          for (int q = 0; q < MAXQ; ++q)
            if (slot[u] != nullptr && q_wc[q] >= 0)  // pad tiles stay 128
              finish(sb[u], q_row0[q], tc[u] * tw4 + q_wc[q], raw[u][q], q_sc[q], q_inv[q]);
      }
    } else {
      for (int t = warp; t < n_tiles; t += kBWarps) {
        const char* slot;
        uint8_t* sb;
        int tc;
        tile_of(t, slot, sb, tc);
        if (slot == nullptr) continue;
        for (int blk = lane; blk < nblk; blk += 32) {
          const Block k = lane_block(U.g, blk, NHB, tc, B.tile_w);
          float sc[NHB], inv[NHB];
          block_scales(k, sc, inv);
          Raw8<SRC> raw[NHB];
          load_block(slot + ((int64_t)k.h0 * U.src.head_stride + k.d0) * ES, raw);
          finish(sb, k.row0, k.wcol, raw, sc, inv);
        }
      }
    }
  }
  __syncthreads();
  // 3. bands -> frames (coalesced rows)
  __shared__ uint8_t* s_row0[16];  // first pixel row of each band (nb <= 16)
  uint8_t* plane = U.fr.base + (int64_t)p * U.fr.plane_stride;
  if (threadIdx.x < nb) {
    const int j = j0 + threadIdx.x;
    const int f = fdiv(B.div_rows, j);
    s_row0[threadIdx.x] = plane + (int64_t)f * U.fr.frame_stride +
                          (int64_t)(j - f * B.grid_rows) * B.tile_h * U.fr.row_pitch;
  }
  __syncthreads();
  const int n_pieces = (nb * B.tile_h) * B.gpr;
  for (int x = threadIdx.x; x < n_pieces; x += kBThreads) {
    const int row_all = fdiv(B.div_gpr, x), piece = x - row_all * B.gpr;
    const int b = row_all >> B.lg_th, r = row_all & (B.tile_h - 1);
    uint8_t* dst = s_row0[b] + (int64_t)r * U.fr.row_pitch;
    const uint8_t* sb = s_band + b * B.band_bytes;
    if (B.g16) {
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        w[e] = *reinterpret_cast<const uint32_t*>(sb + band_word<BD>(B, r, piece * 4 + e));
      st_v4(dst + piece * 16, make_uint4(w[0], w[1], w[2], w[3]));
    } else {
      *reinterpret_cast<uint32_t*>(dst + piece * 4) =
          *reinterpret_cast<const uint32_t*>(sb + band_word<BD>(B, r, piece));
    }
  }
}

bool band_ok(const kvf_plan& p, int32_t dtype, const kvf_surface& fr, const kvf_paged& pg) {
  if (p.b_d >= 8 || p.b_h * p.b_d < 4 || p.D < 8) return false;
  if (dtype != KVF_I8 && p.group_size % 8) return false;
  if (p.frame_w % 4 || fr.row_pitch % 4 || fr.plane_stride % 4 || fr.frame_stride % 4 ||
      reinterpret_cast<uintptr_t>(fr.base) % 4)
    return false;
  const BandGeom b = make_band(p, fr);
  if (b.band_bytes > kBandSmem) return false;
  const int64_t es = (int64_t)dtype_size(dtype);
  const int64_t va = dtype == KVF_I8 ? 8 : 16;
  for (int l = 0; l < 3; ++l)
    if (pg.layer[l] && reinterpret_cast<uintptr_t>(pg.layer[l]) % va) return false;
  if ((pg.head_stride * es) % va || (pg.slot_stride * es) % va || (pg.block_stride * es) % va)
    return false;
  return true;
}

template <int OUT>
void launch_rb(int bd, const RBandParams& P, dim3 grid, size_t smem, cudaStream_t s) {
  switch (bd) {
    case 1: restore_band_kernel<OUT, 1><<<grid, kBThreads, smem, s>>>(P); break;
    case 2: restore_band_kernel<OUT, 2><<<grid, kBThreads, smem, s>>>(P); break;
    default: restore_band_kernel<OUT, 4><<<grid, kBThreads, smem, s>>>(P); break;
  }
}

template <int SRC>
void launch_pb(int bd, const PBandParams& P, dim3 grid, size_t smem, cudaStream_t s) {
  switch (bd) {
    case 1: pack_band_kernel<SRC, 1><<<grid, kBThreads, smem, s>>>(P); break;
    case 2: pack_band_kernel<SRC, 2><<<grid, kBThreads, smem, s>>>(P); break;
    default: pack_band_kernel<SRC, 4><<<grid, kBThreads, smem, s>>>(P); break;
  }
}

}  // namespace

bool restore_band_ok(const kvf_restore_unit& u) {
  return band_ok(u.plan, u.dst.dtype, u.frames, u.dst);
}
bool pack_band_ok(const kvf_pack_unit& u) {
  return band_ok(u.plan, u.src.dtype, u.frames, u.src);
}

// Units sharing (b_d, dtype); launches of up to half KVF_MAX_UNITS units.
kvf_status launch_restore_band(const std::vector<kvf_restore_unit>& units, int32_t dtype,
                               cudaStream_t s) {
  constexpr size_t kPer = KVF_MAX_UNITS / 2;
  for (int bd : {1, 2, 4}) {
    std::vector<const kvf_restore_unit*> mine;
    for (const auto& u : units)
      if (u.plan.b_d == bd) mine.push_back(&u);
    for (size_t at = 0; at < mine.size(); at += kPer) {
      const size_t n = std::min(kPer, mine.size() - at);
      RBandParams* P = new RBandParams();
      P->n_units = (int32_t)n;
      int64_t gx = 0;
      size_t smem = 0;
      for (size_t k = 0; k < n; ++k) {
        const kvf_restore_unit& u = *mine[at + k];
        RBandUnit& d = P->u[k];
        d.fr = u.frames;
        d.g = make_geom(u.plan);
        d.b = make_band(u.plan, u.frames);
        d.scales = u.scales;
        d.dst = u.dst;
        d.div_bs = make_fastdiv(u.dst.block_size);
        d.first_frame = u.first_frame;
        d.n_bands = u.n_frames * u.plan.grid_rows;
        d.G = u.plan.H * u.plan.D / u.plan.group_size;
        gx = std::max<int64_t>(gx, (d.n_bands + d.b.nb - 1) / d.b.nb);
        smem = std::max<size_t>(smem, (size_t)d.b.nb * d.b.band_bytes);
      }
      if (gx > 0) {
        dim3 grid((unsigned)gx, (unsigned)n, 3);
        switch (dtype) {
          case KVF_BF16: launch_rb<KVF_BF16>(bd, *P, grid, smem, s); break;
          case KVF_F16: launch_rb<KVF_F16>(bd, *P, grid, smem, s); break;
          case KVF_F32: launch_rb<KVF_F32>(bd, *P, grid, smem, s); break;
          default: launch_rb<KVF_I8>(bd, *P, grid, smem, s); break;
        }
      }
      delete P;
      KVF_CHECK_CUDA(cudaGetLastError());
    }
  }
  return KVF_OK;
}

// Frames phase of the pack for band units (scales already final in u.scales).
kvf_status launch_pack_band(const std::vector<kvf_pack_unit>& units, int32_t dtype,
                            cudaStream_t s) {
  constexpr size_t kPer = kMaxPackUnits / 2;
  for (int bd : {1, 2, 4}) {
    std::vector<const kvf_pack_unit*> mine;
    for (const auto& u : units)
      if (u.plan.b_d == bd) mine.push_back(&u);
    for (size_t at = 0; at < mine.size(); at += kPer) {
      const size_t n = std::min(kPer, mine.size() - at);
      PBandParams* P = new PBandParams();
      P->n_units = (int32_t)n;
      int64_t gx = 0;
      size_t smem = 0;
      for (size_t k = 0; k < n; ++k) {
        const kvf_pack_unit& u = *mine[at + k];
        PBandUnit& d = P->u[k];
        d.src = u.src;
        d.g = make_geom(u.plan);
        d.b = make_band(u.plan, u.frames);
        d.scales = u.scales;
        d.fr = u.frames;
        d.div_bs = make_fastdiv(u.src.block_size);
        d.n_bands = u.plan.frame_count * u.plan.grid_rows;
        d.G = u.plan.H * u.plan.D / u.plan.group_size;
        gx = std::max<int64_t>(gx, (d.n_bands + d.b.nb - 1) / d.b.nb);
        smem = std::max<size_t>(smem, (size_t)d.b.nb * d.b.band_bytes);
      }
      if (gx > 0) {
        dim3 grid((unsigned)gx, (unsigned)n, 3);
        switch (dtype) {
          case KVF_BF16: launch_pb<KVF_BF16>(bd, *P, grid, smem, s); break;
          case KVF_F16: launch_pb<KVF_F16>(bd, *P, grid, smem, s); break;
          case KVF_F32: launch_pb<KVF_F32>(bd, *P, grid, smem, s); break;
          default: launch_pb<KVF_I8>(bd, *P, grid, smem, s); break;
        }
      }
      delete P;
      KVF_CHECK_CUDA(cudaGetLastError());
    }
  }
  return KVF_OK;
}

}  // namespace kvf
