// kvf_kvfc.cu — KVFC frame-stream decode on the GPU, sm_100a.
//
// 1. rc_decode_kernel: the reference's adaptive range decoder
//    (fk/rangecoder.py:146-189), one thread per (frame, plane) stream — every
//    stream resets its model and is length-prefixed, so they are independent.
//    The per-symbol work is a serial dependency chain, so the kernel is built
//    for latency and few instructions: the model is cumulative counts (block
//    prefix sums in registers, within-block prefix sums as packed u16 in
//    shared memory — 512 B per stream), both searches are 4-level binary
//    searches over registers, the second division is replaced by multiplies,
//    renormalisation is closed-form (clz of low ^ (low + rng)) over a
//    prefetched 64-bit byte window, and a symbol's model update is two 128-bit
//    stores.
// 2. recon_kernel: per-sample prediction (fk/codec.py:131-144) as segmented
//    prefix sums mod 256.  One CTA per chain of same-plane frames starting at
//    an intra frame.  A 16-pixel run of a row never crosses a 16x16 block, so a
//    run is wholly inter (absolute: prev + d) or intra (relative: + d); a warp
//    scans 32 runs at a time with the operator
//      (a, b) -> b.abs ? b : (a.abs, a.v + b.v),
//    after the first column (predicted from above) was scanned down the rows.
#include <algorithm>

#include "kvf_rc_model.cuh"

namespace kvf {
namespace {

using namespace rc;

// Payload bytes through a 64-bit window: `win` holds the 8 bytes at [wa, wa+8),
// the next byte is at `a` with a - wa < 4 at every symbol start.  Positions are
// 32-bit byte offsets from the stream's first aligned word (`org`), so the
// window arithmetic on the decode chain is 32-bit.  A refill shifts in the word
// prefetched one refill earlier (`nxt`), so the load never sits on the decode
// chain; the word is masked as it is shifted in, so every byte of `win` at or
// past the end is already 0 (fk/rangecoder.py:158,181: data[pos] if pos < n)
// and take() needs no bounds test.  Loads use clamped in-bounds addresses.
// FED: the payload is still being copied in (kvf_rc_decode_fed): a word is
// read only once the pieces holding it landed (`ready` pieces of the stream's
// copy segment, acquire).  Pieces end on 128-byte lines, so a line a thread
// caches in L1 never holds bytes that land later.
// FED: what only the landed-bytes poll needs, kept in shared memory (one per
// thread) so that the decode loop carries a single 32-bit bound: with these
// fields live in registers across the loop the FED kernel ran 14% slower.
struct FedCold {
  const uint32_t* ready;  // landed-piece count of the stream's copy segment
  uintptr_t seg0;         // the segment's piece origin (its first 128-byte line)
  uintptr_t org;          // the window's origin
  uint32_t piece;         // piece bytes
  uint32_t pad_;
};

__shared__ FedCold g_fed_cold[kDecThreads];  // FED kernels: one per decoder thread

// Polls until the bytes below offset `need` have landed; returns the landed
// offset (out of line: the decode loop only carries the compare).
__device__ __noinline__ uint32_t fed_poll(uint32_t need) {
  const FedCold* c = &g_fed_cold[threadIdx.x];
  const uintptr_t abs_need = c->org + need;
  for (;;) {
    uint32_t r;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(c->ready) : "memory");
    const uintptr_t av = c->seg0 + (uintptr_t)r * c->piece;
    if (av >= abs_need) {
      const uintptr_t off = av - c->org;
      return off > 0xFFFFFFFFu ? 0xFFFFFFFFu : (uint32_t)off;
    }
    __nanosleep(256);
  }
}

template <bool FED>
struct ByteWindow {
  const uint8_t* org;          // the payload's first byte rounded down to 4
  uint64_t win;
  uint32_t wa, a, end, last;   // offsets from org; last = the last word holding payload
  uint32_t nxt;                // raw word at wa + 8 (loaded one refill ahead)
  uint32_t lim;                // FED: the bytes below offset lim have landed
  __device__ __forceinline__ void await(uint32_t need) {  // bytes below offset need landed
    if (!FED) return;
    need = need < end ? need : end;
    if (need > lim) lim = fed_poll(need);
  }
  // word at offset w with the bytes at or past the end zeroed
  __device__ __forceinline__ uint32_t masked(uint32_t word, uint32_t w) const {
    const int32_t v = (int32_t)(end - w);  // payload bytes in the word
    return v >= 4 ? word : (v <= 0 ? 0u : word & ((1u << (8 * v)) - 1u));
  }
  __device__ __forceinline__ uint32_t load(uint32_t w) {  // clamped in bounds, masked
    const uint32_t x = w < end ? w : last;
    await(x + 4);
    return masked(__ldg(reinterpret_cast<const uint32_t*>(org + x)), w);
  }
  __device__ __forceinline__ void init(const uint8_t* p, uint32_t n) {
    org = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(3));
    a = (uint32_t)(p - org);
    end = a + n;
    wa = 0;
    last = n ? (end - 1) & ~3u : 0u;
    if (n == 0) {  // every byte reads as 0; never dereference
      win = 0;
      nxt = 0;
      end = 0;
      return;
    }
    win = (uint64_t)load(0) | ((uint64_t)load(4) << 32);
    nxt = load(8) ;
  }
  __device__ __forceinline__ uint32_t peek() const {  // byte at a (a - wa < 8)
    return (uint32_t)(win >> (8 * (a - wa))) & 0xFFu;
  }
  // The next n <= 3 bytes as a big-endian number (first byte most significant;
  // bytes at or past the end are 0); advances a.  Needs a - wa < 4.
  __device__ __forceinline__ uint32_t take(uint32_t n) {
    const uint32_t w = (uint32_t)(win >> (8 * (a - wa)));  // bytes a.. a+3, little-endian
    const uint32_t be = __byte_perm(w, 0u, 0x0123);         // byte a in bits 24..31
    a += n;
    return n ? be >> (32 - 8 * n) : 0u;
  }
  // Keep a - wa < 4: shift in the prefetched word (masked only now, so the
  // load it came from had a whole symbol to land) and prefetch the next one.
  __device__ __forceinline__ void refill() {
    const bool go = a - wa >= 4;
    const uint64_t shifted = (win >> 32) | ((uint64_t)masked(nxt, wa + 8) << 32);
    win = go ? shifted : win;
    wa = go ? wa + 4 : wa;
    // predicated load straight into `nxt`: no instruction consumes it until
    // the next refill, so its latency never stalls the decode chain
    const uint32_t x = wa + 8 < end ? wa + 8 : last;
    const uint8_t* src = org + x;
    // (FED: the block-level wait of rc_decode_kernel covers this prefetch)
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p ld.global.nc.u32 %0, [%1];\n}"
        : "+r"(nxt)
        : "l"(src), "r"((uint32_t)(go && end != 0)));
    // When that word starts a 128-byte line, pull the line two ahead into L1:
    // otherwise the first load of each line misses to DRAM, longer than one
    // symbol, and the next refill waits for it (8% of the decode's stalls).
    // FED: only a line that has wholly landed (below lim; pieces end on lines),
    // so L1 never holds bytes that land later.
    const bool line = go && ((uint32_t)reinterpret_cast<uintptr_t>(src) & 127u) == 0 &&
                      (FED ? x + 384 <= lim : x + 256 < end);
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.u32 p, %1, 0;\n @p prefetch.global.L1 [%0];\n}"
        :: "l"(src + 256), "r"((uint32_t)line));
  }
};

#ifdef KVF_TRACE
// trace builds (tools/trace_fed.py): globaltimer per stream [start, first
// bytes, done] and per copy CTA [done]
__device__ unsigned long long* g_fed_trace;
__device__ __forceinline__ void fed_mark(int i, int e) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (g_fed_trace) g_fed_trace[(size_t)i * 4 + e] = t;
}
#else
__device__ __forceinline__ void fed_mark(int, int) {}
#endif

// The copy side of kvf_rc_decode_fed: CTAs [0, n_copy) move the segments
// host -> device over PCIe (16-byte loads of mapped pinned memory), piece r of
// every segment before piece r+1 of any, and count each segment's landed
// pieces in ready[] (in order, release).
// symbols decoded per landed-bytes check: 64 needs 528 bytes landed ahead (128
// and 256 made the decoders wait near the copy frontier: 199 / 286 ms on C2)
constexpr uint32_t kFedBlock = 64;

struct FeedArgs {
  const kvf_feed_seg* segs;
  const int32_t* seg_of;  // stream -> segment
  uint32_t* ready;
  int32_t n_segs, n_copy, piece, rounds;
};

__device__ void copy_pieces(const FeedArgs& F) {
  const int lane = threadIdx.x;
  const int64_t n_t = (int64_t)F.rounds * F.n_segs;
  for (int64_t t = blockIdx.x; t < n_t; t += F.n_copy) {
    const int r = (int)(t / F.n_segs), k = (int)(t - (int64_t)r * F.n_segs);
    const kvf_feed_seg sg = F.segs[k];
    // piece r = the segment's bytes in [L0 + r P, L0 + (r+1) P), L0 = its
    // first 128-byte line: piece ends fall on line boundaries
    const int64_t head0 = (int64_t)(reinterpret_cast<uintptr_t>(sg.dst) & 127);
    const int64_t lo = max((int64_t)0, (int64_t)r * F.piece - head0);
    const int64_t hi = min(sg.len, (int64_t)(r + 1) * F.piece - head0);
    if (lo >= hi) continue;
    const uint8_t* src = sg.src + lo;
    uint8_t* dst = sg.dst + lo;
    const int64_t n = hi - lo;
    // bytes up to 16-aligned dst, then 16-byte vectors when src is aligned alike
    const int64_t head = min(n, (int64_t)((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15));
    for (int64_t e = lane; e < head; e += 32) dst[e] = src[e];
    const bool vec = ((reinterpret_cast<uintptr_t>(src + head) & 15) == 0);
    const int64_t nv = vec ? (n - head) / 16 : 0;
    const uint4* s4 = reinterpret_cast<const uint4*>(src + head);
    uint4* d4 = reinterpret_cast<uint4*>(dst + head);
#pragma unroll 4
    for (int64_t e = lane; e < nv; e += 32) d4[e] = ld_nc_v4(s4 + e);
    for (int64_t e = head + nv * 16 + lane; e < n; e += 32) dst[e] = src[e];
    __threadfence();  // this lane's bytes before the count
    __syncwarp();
    if (lane == 0) {
      uint32_t* rd = F.ready + k;
      uint32_t cur;
      do {  // piece r - 1 of this segment (an earlier ticket) counted first
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(rd) : "memory");
      } while (cur != (uint32_t)r);
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(rd), "r"((uint32_t)r + 1) : "memory");
    }
  }
}

// EVERY: every symbol stores its 4-symbol group's word (no branch on k & 3):
// one more instruction per symbol, faster while each scheduler holds at most
// one decoder warp (latency-bound: C2 R1080 93.7 -> 92.0 ms), slower once
// warps share schedulers (issue-bound: C2 R240 22.1 -> 27.9 ms) and in the fed
// kernel (95.4 -> 98.4 ms).
template <bool FED, bool EVERY = false>
__global__ void __launch_bounds__(kDecThreads)
    rc_decode_kernel(const kvf_rc_stream* __restrict__ streams, int n, const FeedArgs F) {
  extern __shared__ uint4 M[];  // [32 chunks][kDecThreads] x 16 B
  __shared__ uint4 T_add[2 * kAddRows];  // increment rows (rc::add_table_init)
  if (FED && (int)blockIdx.x < F.n_copy) {
    copy_pieces(F);
    if (threadIdx.x == 0) fed_mark(n + blockIdx.x, 3);
    return;
  }
  add_table_init(T_add);       // the whole warp, before any thread leaves
  const int tid = threadIdx.x;
  const int sidx = ((int)blockIdx.x - (FED ? F.n_copy : 0)) * kDecThreads + tid;
  const unsigned live = __ballot_sync(0xffffffffu, sidx < n);  // the warp's streams
  if (sidx >= n) return;
  const kvf_rc_stream st = streams[sidx];
  uint4* m = M + tid;  // chunk c of this thread's model at m[c * kDecThreads]
  uint32_t P[8];       // block prefixes CB[2w] | CB[2w+1] << 16
  model_init(m, P);
  uint32_t total = 256, low = 0, rng = 0xFFFFFFFFu, code = 0;
  ByteWindow<FED> bw;
  if constexpr (FED) {
    const int k = F.seg_of[sidx];
    FedCold& c = g_fed_cold[tid];
    c.seg0 = reinterpret_cast<uintptr_t>(F.segs[k].dst) & ~uintptr_t(127);  // piece origin
    c.piece = (uint32_t)F.piece;
    c.ready = F.ready + k;
    c.org = reinterpret_cast<uintptr_t>(st.payload) & ~uintptr_t(3);  // = bw.org (init)
    bw.lim = 0;
  }
  if (FED) fed_mark(sidx, 0);
  bw.init(st.payload, (uint32_t)st.len);
  // FED: the warp's 32 streams start together once each has its first bytes.
  // A thread that started alone would run its whole decode loop while the
  // warp's waiting threads are never scheduled (divergent paths serialise).
  if (FED) __syncwarp(live);
  if (FED) fed_mark(sidx, 1);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    code = (code << 8) | bw.peek();
    ++bw.a;
  }
  bw.refill();

  uint8_t* out = st.symbols;
  const uint32_t nsym = (uint32_t)st.n_symbols;
  uint32_t pack = 0;
  const bool aligned4 = (reinterpret_cast<uintptr_t>(out) & 3) == 0;
  const uint32_t full4 = nsym & ~3u;  // symbols in whole 4-symbol groups
  float rcp = rcp_approx(total);  // ~1/total of the symbol being decoded
  // FED: blocks of kFedBlock symbols, each started only once the next
  // kFedBlock * 8 + 16 payload bytes have landed.  A symbol takes at most 7
  // bytes (at most 3 in the closed-form shift, then rng >= 1 needs at most 3
  // more shifts to reach 2^24, where the top bytes of low and low + rng always
  // differ, fk/rangecoder.py:171-183) and the window prefetch reads 12 bytes
  // ahead, so no read inside a block passes the landed bytes.
  for (uint32_t k0 = 0; k0 < nsym; k0 += kFedBlock) {
  if (FED) bw.await(bw.a + kFedBlock * 8 + 16);
  const uint32_t k1 = min(nsym, k0 + kFedBlock);
  for (uint32_t k = k0; k < k1; ++k) {
    const float rcp_next = rcp_approx(total + kInc);  // off the chain
    const uint32_t r = exact_div(rng, total, rcp);  // rng / total (fk/rangecoder.py:163)
    // Largest s with cum(s) <= min((code - low) / r, total - 1) (fk/rangecoder.py:
    // 163-166, 79-90) without the second division: cum <= x / r <=> cum * r <= x.
    // cum is increasing in s, so both searches are binary over registers.
    const uint32_t x = code - low;
    // block: largest b with CB[b] * r <= x (CB[0] = 0 always qualifies)
    // The level-i operand is CB[(bits above) | 2^i]; CB[blk] is the operand of
    // the last level that compared true (CB[0] = 0 if none), so `base` is a
    // 4-select chain that finishes one select after b0.
    // (CB[2w] is the low and CB[2w+1] the high half of P[w]; the selects pick
    // packed words, levels 3..1 read low halves, level 0 a high half)
    const uint32_t o3 = cb_lo(P[4]);                               // CB[8]
    const bool b3 = o3 * r <= x;
    const uint32_t o2 = cb_lo(b3 ? P[6] : P[2]);                   // CB[12] : CB[4]
    const bool b2 = o2 * r <= x;
    const uint32_t w2a = b3 ? P[5] : P[1], w2b = b3 ? P[7] : P[3];  // CB[10|2], CB[14|6]
    const uint32_t o1 = cb_lo(b2 ? w2b : w2a);
    const bool b1 = o1 * r <= x;
    const uint32_t w1a = b3 ? P[4] : P[0], w1c = b3 ? P[6] : P[2];  // CB[9|1], CB[13|5]
    const uint32_t w1e = b2 ? w1c : w1a, w1f = b2 ? w2b : w2a;       // (+ CB[11|3|15|7])
    const uint32_t o0 = cb_hi(b1 ? w1f : w1e);
    const bool b0 = o0 * r <= x;
    const uint32_t blk = (b3 ? 8u : 0u) + (b2 ? 4u : 0u) + (b1 ? 2u : 0u) + (b0 ? 1u : 0u);
    uint32_t base = b3 ? o3 : 0u;
    base = b2 ? o2 : base;
    base = b1 ? o1 : base;
    base = b0 ? o0 : base;
    const uint4 cbi[2] = {T_add[2 * (blk + 1)], T_add[2 * (blk + 1) + 1]};  // CB[q>blk] += INC
    const uint32_t rem = x - base * r;
    // within the block: incl[0..15] from two 128-bit loads
    const uint4 ca = m[(2 * blk) * kDecThreads], cb = m[(2 * blk + 1) * kDecThreads];
    const uint32_t wv[8] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
    // sl = number of j in 0..14 with incl[j] * r <= rem; lo/hi = incl[sl-1] (or 0), incl[sl]
    const uint32_t i7 = hi16(wv[3]);
    const bool t3 = i7 * r <= rem;
    const uint32_t i3 = t3 ? hi16(wv[5]) : hi16(wv[1]);   // incl[11] : incl[3]
    const bool t2 = i3 * r <= rem;
    uint32_t i1;
    {
      const uint32_t a = t3 ? hi16(wv[4]) : hi16(wv[0]);  // incl[9] : incl[1]
      const uint32_t b = t3 ? hi16(wv[6]) : hi16(wv[2]);  // incl[13] : incl[5]
      i1 = t2 ? b : a;
    }
    const bool t1 = i1 * r <= rem;
    uint32_t i0, lo_v, hi_v;
    {
      // candidates for incl[sl'] with sl' = 8t3 + 4t2 + 2t1 (+ 0 / + 1)
      const uint32_t q0 = t3 ? wv[4] : wv[0], q1 = t3 ? wv[5] : wv[1];
      const uint32_t q2 = t3 ? wv[6] : wv[2], q3 = t3 ? wv[7] : wv[3];
      const uint32_t p0 = t2 ? q2 : q0, p1 = t2 ? q3 : q1;
      const uint32_t pair = t1 ? p1 : p0;  // incl[sl'] | incl[sl' + 1] << 16
      i0 = lo16(pair);
      const bool t0 = i0 * r <= rem;
      // incl[sl' - 1] (0 at sl' = 0) is the operand of the last of levels 3..1
      // that compared true, as for `base`
      uint32_t below = t3 ? i7 : 0u;
      below = t2 ? i3 : below;
      below = t1 ? i1 : below;
      lo_v = t0 ? i0 : below;
      hi_v = t0 ? hi16(pair) : i0;
      const uint32_t sl = (t3 ? 8u : 0u) + (t2 ? 4u : 0u) + (t1 ? 2u : 0u) + (t0 ? 1u : 0u);
      const uint32_t s = 16u * blk + sl;
      // state update (fk/rangecoder.py:168-170)
      low = code - (rem - lo_v * r);                       // low + r * cum(s)
      rng = r * (hi_v - lo_v);                             // r * freq(s)
      // renormalise (fk/rangecoder.py:171-183).  While the top byte of low and
      // low + rng agree the reference shifts a byte in; shifting both by 8
      // shifts X = low ^ (low + rng) by 8, so that phase is exactly
      // n = clz(X) / 8 bytes (rng >= 1, so X != 0 and n <= 3).  Only if rng
      // is then below 2^16 does the squeeze branch run (rare): the loop below
      // replays the reference rounds from there.
      {
        const uint32_t n = __clz(low ^ (low + rng)) >> 3;
        const uint32_t bytes = bw.take(n);  // the next n bytes, big-endian, in the low bits
        code = n ? (code << (8 * n)) | bytes : code;
        low = n ? low << (8 * n) : low;
        rng = n ? rng << (8 * n) : rng;
      }
      bw.refill();
      while (rng < kBot || (low ^ (low + rng)) < kTop) {
        if ((low ^ (low + rng)) >= kTop) rng = (0u - low) & (kBot - 1);
        code = (code << 8) | bw.take(1);
        low <<= 8;
        rng <<= 8;
        bw.refill();
      }
      pack = (pack >> 8) | (s << 24);  // 4 symbols per 32-bit word
      if (EVERY && aligned4 && k < full4) {
        // the group's last symbol stores the complete word last
        *reinterpret_cast<uint32_t*>(out + (k & ~3u)) = pack;
      } else if ((k & 3) == 3) {
        if (aligned4) {
          *reinterpret_cast<uint32_t*>(out + (k - 3)) = pack;
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) out[k - 3 + e] = (uint8_t)(pack >> (8 * e));
        }
      }
      model_update(m, P, blk, sl, wv, T_add, cbi);  // fk/rangecoder.py:185-186
    }
    total += kInc;
    rcp = rcp_next;
    if (total >= kLimit) {
      total = rebuild(m, P);
      rcp = rcp_approx(total);
    }
  }
  }
  if (nsym & 3) {  // tail: the last nsym % 4 symbols sit in the top bytes of `pack`
    const uint32_t base = nsym & ~3u, n_tail = nsym & 3;
    for (uint32_t k = base; k < nsym; ++k) out[k] = (uint8_t)(pack >> (8 * (4 - n_tail + k - base)));
  }
  if (FED) fed_mark(sidx, 2);
}

// ----------------------------------------------------------- reconstruction
struct Seg {
  uint32_t abs;  // 1 = value is absolute
  uint32_t v;    // value (abs) or increment (relative), mod 256 in the low byte
};

__device__ __forceinline__ Seg seg_combine(Seg a, Seg b) {
  return b.abs ? b : Seg{a.abs, a.v + b.v};
}

// Inclusive warp scan of Seg; returns the inclusive value for this lane.
__device__ __forceinline__ Seg warp_seg_scan(Seg x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Seg y;
    y.abs = __shfl_up_sync(0xffffffffu, x.abs, o);
    y.v = __shfl_up_sync(0xffffffffu, x.v, o);
    if (lane >= o) x = seg_combine(y, x);
  }
  return x;
}

__device__ __forceinline__ int unzig(uint32_t z) {
  return (z & 1) ? -(int)((z + 1) >> 1) : (int)(z >> 1);
}

__device__ __forceinline__ bool mode_bit(const uint8_t* modes, int bw, int by, int bx) {
  if (!modes) return false;
  const int b = by * bw + bx;
  return (modes[b >> 3] >> (7 - (b & 7))) & 1;  // np.packbits: MSB first
}

constexpr int kReconThreads = 128;

// ---- byte-lane (SWAR) helpers: four samples per 32-bit word, mod 256
__device__ __forceinline__ uint32_t add_bytes(uint32_t a, uint32_t b) {
  return ((a & 0x7F7F7F7Fu) + (b & 0x7F7F7F7Fu)) ^ ((a ^ b) & 0x80808080u);
}
__device__ __forceinline__ uint32_t unzig_bytes(uint32_t z) {  // per byte: (z>>1) ^ -(z&1)
  return ((z >> 1) & 0x7F7F7F7Fu) ^ ((z & 0x01010101u) * 0xFFu);
}
__device__ __forceinline__ uint32_t bcast_byte(uint32_t b) { return (b & 0xFFu) * 0x01010101u; }
// inclusive prefix sums mod 256 over the 16 bytes of q (byte 0 first)
__device__ __forceinline__ uint4 prefix_bytes16(uint4 q) {
  q.x = add_bytes(q.x, q.x << 8);
  q.x = add_bytes(q.x, q.x << 16);
  q.y = add_bytes(q.y, q.y << 8);
  q.y = add_bytes(q.y, q.y << 16);
  q.z = add_bytes(q.z, q.z << 8);
  q.z = add_bytes(q.z, q.z << 16);
  q.w = add_bytes(q.w, q.w << 8);
  q.w = add_bytes(q.w, q.w << 16);
  q.y = add_bytes(q.y, bcast_byte(q.x >> 24));
  q.z = add_bytes(q.z, bcast_byte(q.y >> 24));
  q.w = add_bytes(q.w, bcast_byte(q.z >> 24));
  return q;
}

// One row of a plane, 16 samples per lane and 512 per warp step, when rows
// are 16-B aligned and the width is a multiple of 16: vector loads/stores,
// the next step's loads in flight while this step scans.  Column 0 (phase
// A) is the row's initial carry; its symbol is dropped from an intra run.
__device__ __forceinline__ void recon_row_vec(const uint8_t* sym, const uint8_t* prow,
                                              uint8_t* orow, const uint8_t* modes, int bw,
                                              int by, int w, uint32_t carry) {
  const int lane = threadIdx.x & 31;
  auto load = [&](int x0, uint4& sv, uint4& pv, bool& inter) {
    const int xs = x0 + lane * 16;
    sv = make_uint4(0u, 0u, 0u, 0u);
    pv = sv;
    inter = false;
    if (xs < w) {
      sv = __ldg(reinterpret_cast<const uint4*>(sym + xs));
      inter = mode_bit(modes, bw, by, xs >> 4);
      if (prow) pv = __ldcg(reinterpret_cast<const uint4*>(prow + xs));
    }
  };
  uint4 sv, pv;
  bool inter;
  load(0, sv, pv, inter);
  for (int x0 = 0; x0 < w; x0 += 32 * 16) {
    uint4 sn, pn;
    bool in_n;
    load(x0 + 32 * 16, sn, pn, in_n);
    const int xs = x0 + lane * 16;
    uint4 d = make_uint4(unzig_bytes(sv.x), unzig_bytes(sv.y), unzig_bytes(sv.z),
                         unzig_bytes(sv.w));
    uint4 v;
    Seg run;
    if (inter) {
      v = make_uint4(add_bytes(pv.x, d.x), add_bytes(pv.y, d.y), add_bytes(pv.z, d.z),
                     add_bytes(pv.w, d.w));
      run = Seg{1u, v.w >> 24};
    } else {
      if (xs == 0) d.x &= 0xFFFFFF00u;  // sample 0 = carry (phase A)
      v = prefix_bytes16(d);
      run = Seg{0u, v.w >> 24};
    }
    if (xs >= w) run = Seg{0u, 0u};
    const Seg inc = warp_seg_scan(run);
    Seg exc;
    exc.abs = __shfl_up_sync(0xffffffffu, inc.abs, 1);
    exc.v = __shfl_up_sync(0xffffffffu, inc.v, 1);
    const uint32_t before = lane > 0 ? (exc.abs ? exc.v : carry + exc.v) : carry;
    if (!inter) {
      const uint32_t b = bcast_byte(before);
      v = make_uint4(add_bytes(v.x, b), add_bytes(v.y, b), add_bytes(v.z, b), add_bytes(v.w, b));
    }
    if (xs < w) *reinterpret_cast<uint4*>(orow + xs) = v;
    const uint32_t last = inc.abs ? inc.v : carry + inc.v;
    carry = __shfl_sync(0xffffffffu, last, 31);
    sv = sn;
    pv = pn;
    inter = in_n;
  }
}

__device__ __forceinline__ bool al16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

__global__ void __launch_bounds__(kReconThreads)
    recon_kernel(const kvf_recon_plane* __restrict__ planes,
                 const kvf_recon_chain* __restrict__ chains) {
  const kvf_recon_chain ch = chains[blockIdx.x];
  const int h = ch.height, w = ch.width;
  const int bw = (w + 15) / 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  for (int e = 0; e < ch.count; ++e) {
    const kvf_recon_plane P = planes[ch.first + e];
    if (P.symbols == nullptr) continue;  // reconstructed earlier: only a reference
    const uint8_t* prev = e > 0 ? planes[ch.first + e - 1].out : nullptr;
    const int64_t prev_pitch = e > 0 ? planes[ch.first + e - 1].out_pitch : 0;
    const uint8_t* modes = e > 0 ? P.modes : nullptr;
    // Phase A: first column, scanned down the rows by warp 0 (carry starts at
    // the corner prediction 128).
    if (warp == 0) {
      uint32_t carry = 128;
      for (int y0 = 0; y0 < h; y0 += 32) {
        const int y = y0 + lane;
        Seg x{0u, 0u};
        if (y < h) {
          const int d = unzig(P.symbols[(int64_t)y * w]);
          if (mode_bit(modes, bw, y >> 4, 0))
            x = Seg{1u, (uint32_t)(prev[(int64_t)y * prev_pitch] + d)};
          else
            x = Seg{0u, (uint32_t)d};
        }
        Seg inc = warp_seg_scan(x);
        const uint32_t val = inc.abs ? inc.v : carry + inc.v;
        if (y < h) P.out[(int64_t)y * P.out_pitch] = (uint8_t)val;
        carry = __shfl_sync(0xffffffffu, val, 31);
      }
    }
    __syncthreads();
    // Phase B: each warp scans whole rows in spans of 32 runs x 16 pixels.
    const bool vec = (w & 15) == 0 && al16(P.symbols) && al16(P.out) && (P.out_pitch & 15) == 0 &&
                     (prev == nullptr || (al16(prev) && (prev_pitch & 15) == 0));
    if (vec) {
      for (int y = warp; y < h; y += nwarps) {
        uint8_t* orow = P.out + (int64_t)y * P.out_pitch;
        recon_row_vec(P.symbols + (int64_t)y * w, prev ? prev + (int64_t)y * prev_pitch : nullptr,
                      orow, modes, bw, y >> 4, w, orow[0]);
      }
      __syncthreads();
      continue;
    }
    for (int y = warp; y < h; y += nwarps) {
      const uint8_t* sym = P.symbols + (int64_t)y * w;
      uint8_t* orow = P.out + (int64_t)y * P.out_pitch;
      const uint8_t* prow = prev ? prev + (int64_t)y * prev_pitch : nullptr;
      uint32_t carry = orow[0];  // column 0 from phase A
      for (int x0 = 0; x0 < w; x0 += 32 * 16) {
        const int xs = x0 + lane * 16;
        const int nrun = max(0, min(16, w - xs));
        const bool inter = nrun > 0 && mode_bit(modes, bw, y >> 4, xs >> 4);
        uint8_t vals[16];
        Seg run{0u, 0u};
        for (int k = 0; k < nrun; ++k) {
          const int x = xs + k;
          const int d = unzig(sym[x]);
          if (x == 0) {
            vals[k] = (uint8_t)carry;  // already final
            run = Seg{1u, carry};
          } else if (inter) {
            vals[k] = (uint8_t)(prow[x] + d);
            run = Seg{1u, vals[k]};
          } else {
            vals[k] = (uint8_t)d;  // relative increment for now
            run = seg_combine(run, Seg{0u, (uint32_t)d});
          }
        }
        const Seg inc = warp_seg_scan(run);
        // exclusive prefix = value just before this run
        Seg exc;
        exc.abs = __shfl_up_sync(0xffffffffu, inc.abs, 1);
        exc.v = __shfl_up_sync(0xffffffffu, inc.v, 1);
        uint32_t before = carry;
        if (lane > 0) before = exc.abs ? exc.v : carry + exc.v;
        if (!inter) {
          uint32_t acc = before;
          for (int k = 0; k < nrun; ++k) {
            if (xs + k == 0) {
              acc = carry;
              continue;
            }
            acc += vals[k];
            vals[k] = (uint8_t)acc;
          }
        }
        for (int k = 0; k < nrun; ++k) orow[xs + k] = vals[k];
        const uint32_t last = inc.abs ? inc.v : carry + inc.v;
        carry = __shfl_sync(0xffffffffu, last, 31);
      }
    }
    __syncthreads();  // frame e complete before e+1 predicts from it
  }
}

}  // namespace
}  // namespace kvf

using namespace kvf;

extern "C" kvf_status kvf_rc_decode(const kvf_rc_stream* d_streams, int32_t n_streams,
                                    void* stream) {
  if (n_streams < 0 || (n_streams > 0 && !d_streams)) KVF_FAIL(KVF_EINVAL, "bad stream array");
  if (n_streams == 0) return KVF_OK;
  // One warp per CTA; its 32 models take 16 KB of shared memory, so fourteen
  // CTAs (448 streams) are resident per SM and the grid spreads over every SM.
  const size_t smem = (size_t)kDecThreads * 256 * sizeof(uint16_t);
  const int grid = (n_streams + kDecThreads - 1) / kDecThreads;
  int dev = 0, sms = 0;
  KVF_CHECK_CUDA(cudaGetDevice(&dev));
  KVF_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  FeedArgs none{};
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // few enough warps that a scheduler rarely holds two, even when a few such
  // launches (decode_batch parts) run side by side
  if (grid <= 2 * sms)
    rc_decode_kernel<false, true><<<grid, kDecThreads, smem, s>>>(d_streams, n_streams, none);
  else
    rc_decode_kernel<false, false><<<grid, kDecThreads, smem, s>>>(d_streams, n_streams, none);
  KVF_CHECK_CUDA(cudaGetLastError());
  return KVF_OK;
}

extern "C" kvf_status kvf_rc_decode_fed(const kvf_rc_stream* d_streams, int32_t n_streams,
                                        const kvf_feed_seg* d_segs, const int32_t* d_seg_of,
                                        int32_t n_segs, int32_t piece_bytes, int64_t max_seg_len,
                                        uint32_t* ready, int32_t n_copy_ctas, void* stream) {
  if (n_streams < 0 || n_segs < 0 || (n_streams > 0 && (!d_streams || !d_seg_of)) ||
      (n_segs > 0 && (!d_segs || !ready)))
    KVF_FAIL(KVF_EINVAL, "bad stream / segment arrays");
  if (piece_bytes < 256 || piece_bytes % 128 || n_copy_ctas < 1 || max_seg_len < 0)
    KVF_FAIL(KVF_EINVAL, "bad piece size / copy CTA count");
  if (n_streams == 0 && n_segs == 0) return KVF_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (n_segs) KVF_CHECK_CUDA(cudaMemsetAsync(ready, 0, sizeof(uint32_t) * n_segs, s));
  const int grid = n_copy_ctas + (n_streams + kDecThreads - 1) / kDecThreads;
  // every CTA co-resident (decoders wait on copiers): a cooperative launch.
  // The shared memory request spreads the CTAs over the SMs (a cooperative
  // grid is packed; serial decode chains sharing a scheduler slow each other)
  int dev = 0, sms = 0, per_sm = 0, smem_sm = 0;
  KVF_CHECK_CUDA(cudaGetDevice(&dev));
  KVF_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  KVF_CHECK_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
  const int want_per_sm = std::max(1, (grid + sms - 1) / sms);
  cudaFuncAttributes fa{};
  KVF_CHECK_CUDA(cudaFuncGetAttributes(&fa, rc_decode_kernel<true>));
  // per CTA: dynamic + static shared memory + the 1 KB the hardware reserves
  size_t smem = (size_t)kDecThreads * 256 * sizeof(uint16_t);
  smem = std::max(smem, (size_t)(smem_sm / want_per_sm) - fa.sharedSizeBytes - 1024 - 512);
  smem = std::min<size_t>(smem, 200 * 1024);
  KVF_CHECK_CUDA(cudaFuncSetAttribute(rc_decode_kernel<true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  KVF_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rc_decode_kernel<true>,
                                                               kDecThreads, smem));
  if ((int64_t)per_sm * sms < grid)
    KVF_FAIL(KVF_EUNSUPPORTED, "fed decode of %d streams does not fit one wave", n_streams);
  FeedArgs F;
  F.segs = d_segs;
  F.seg_of = d_seg_of;
  F.ready = ready;
  F.n_segs = n_segs;
  F.n_copy = n_copy_ctas;
  F.piece = piece_bytes;
  F.rounds = (int32_t)((max_seg_len + 127 + piece_bytes - 1) / piece_bytes);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kDecThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  KVF_CHECK_CUDA(cudaLaunchKernelEx(&cfg, rc_decode_kernel<true>, d_streams, (int)n_streams, F));
  return KVF_OK;
}

extern "C" kvf_status kvf_kvfc_reconstruct(const kvf_recon_plane* d_planes,
                                           const kvf_recon_chain* d_chains, int32_t n_chains,
                                           void* stream) {
  if (n_chains < 0 || (n_chains > 0 && (!d_planes || !d_chains)))
    KVF_FAIL(KVF_EINVAL, "bad chain arrays");
  if (n_chains == 0) return KVF_OK;
  recon_kernel<<<n_chains, kReconThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(d_planes,
                                                                                     d_chains);
  KVF_CHECK_CUDA(cudaGetLastError());
  return KVF_OK;
}

#ifdef KVF_TRACE
extern "C" int kvf_fed_trace_set(void* p) {
  return (int)cudaMemcpyToSymbol(kvf::g_fed_trace, &p, sizeof(p));
}
#endif
