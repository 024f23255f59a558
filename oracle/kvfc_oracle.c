/*
 * kvfc_oracle.c — CPU restatement of the reference KVFC entropy coder and
 * predictor.  TEST INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg as the checker / CPU baseline; never linked
 * into the product library.
 *
 * Restates (pinned against golden vectors generated from the reference):
 *   - adaptive order-0 model: 256 symbols, counts start at 1, +INC=32 per coded
 *     symbol, all counts halved ((c+1)>>1) once total >= 2^16
 *     (fk/rangecoder.py:44-103)
 *   - carry-less 32-bit range coder with the 2^16 squeeze
 *     (fk/rangecoder.py:106-143 encode, :146-189 decode; 4 flush bytes,
 *     reads past the end yield 0)
 *   - per-pixel reconstruction: inter = co-located previous-frame sample,
 *     intra = left, first column from above, corner from 128
 *     (fk/codec.py:131-144)
 * The cumulative counts use a plain array walk instead of the reference's
 * Fenwick tree: identical arithmetic, simpler code.
 */
#include <stdint.h>
#include <string.h>

#define ALPHA 256
#define INC 32u
#define LIMIT (1u << 16)
#define TOP (1u << 24)
#define BOT (1u << 16)

typedef struct {
  uint32_t freq[ALPHA];
  uint32_t total;
} model_t;

static void model_init(model_t* m) {
  for (int i = 0; i < ALPHA; ++i) m->freq[i] = 1;
  m->total = ALPHA;
}

static void model_update(model_t* m, int s) {
  m->freq[s] += INC;
  m->total += INC;
  if (m->total >= LIMIT) {
    uint32_t t = 0;
    for (int i = 0; i < ALPHA; ++i) {
      m->freq[i] = (m->freq[i] + 1) >> 1;
      t += m->freq[i];
    }
    m->total = t;
  }
}

static uint32_t cum_below(const model_t* m, int s) {
  uint32_t c = 0;
  for (int i = 0; i < s; ++i) c += m->freq[i];
  return c;
}

int64_t kvfo_rc_encode(const uint8_t* sym, int64_t n, uint8_t* out) {
  model_t m;
  model_init(&m);
  uint32_t low = 0, rng = 0xFFFFFFFFu;
  int64_t k = 0;
  for (int64_t i = 0; i < n; ++i) {
    int s = sym[i];
    uint32_t r = rng / m.total;
    low += r * cum_below(&m, s);
    rng = r * m.freq[s];
    for (;;) {
      if ((low ^ (low + rng)) >= TOP) {
        if (rng >= BOT) break;
        rng = (0u - low) & (BOT - 1);
      }
      out[k++] = (uint8_t)(low >> 24);
      low <<= 8;
      rng <<= 8;
    }
    model_update(&m, s);
  }
  for (int j = 0; j < 4; ++j) {
    out[k++] = (uint8_t)(low >> 24);
    low <<= 8;
  }
  return k;
}

void kvfo_rc_decode(const uint8_t* data, int64_t n_data, int64_t n_sym, uint8_t* out) {
  model_t m;
  model_init(&m);
  uint32_t low = 0, rng = 0xFFFFFFFFu, code = 0;
  int64_t pos = 0;
  for (int j = 0; j < 4; ++j, ++pos) code = (code << 8) | (pos < n_data ? data[pos] : 0u);
  for (int64_t i = 0; i < n_sym; ++i) {
    uint32_t r = rng / m.total;
    uint32_t v = (code - low) / r;
    if (v >= m.total) v = m.total - 1;
    int s = 0;
    uint32_t c = 0;
    while (c + m.freq[s] <= v) c += m.freq[s++];
    low += r * c;
    rng = r * m.freq[s];
    for (;;) {
      if ((low ^ (low + rng)) >= TOP) {
        if (rng >= BOT) break;
        rng = (0u - low) & (BOT - 1);
      }
      code = (code << 8) | (pos < n_data ? data[pos] : 0u);
      ++pos;
      low <<= 8;
      rng <<= 8;
    }
    out[i] = (uint8_t)s;
    model_update(&m, s);
  }
}

/* symbols: zigzag symbols [h*w]; modes: [ceil(h/16) * ceil(w/16)] (1 = inter);
 * prev: previous frame plane (read only where use_inter && mode == 1). */
void kvfo_reconstruct_plane(const uint8_t* symbols, const uint8_t* modes,
                            const uint8_t* prev, int use_inter, int h, int w,
                            uint8_t* plane) {
  const int bw = (w + 15) / 16;
  for (int y = 0; y < h; ++y) {
    for (int x = 0; x < w; ++x) {
      int z = symbols[(int64_t)y * w + x];
      int d = (z & 1) ? -((z + 1) >> 1) : (z >> 1); /* un-zigzag */
      int pred;
      if (use_inter && modes[(y >> 4) * bw + (x >> 4)] == 1)
        pred = prev[(int64_t)y * w + x];
      else if (x > 0)
        pred = plane[(int64_t)y * w + x - 1];
      else if (y > 0)
        pred = plane[(int64_t)(y - 1) * w];
      else
        pred = 128;
      plane[(int64_t)y * w + x] = (uint8_t)((pred + d) & 0xFF);
    }
  }
}
