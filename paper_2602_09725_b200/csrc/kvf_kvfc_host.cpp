// kvf_kvfc_host.cpp — host walk of a KVFC frame stream (no entropy decoding).
//
// Stream layout (fk/codec.py:16-20, little-endian):
//   u32 frame_count, u32 height, u32 width
//   per frame: u8 frame_type (0 intra, 1 inter)
//     per plane (3): [inter only: packed mode bitmap, ceil(bh*bw/8) bytes]
//                    u32 payload length, payload
// The walk raises (KVF_EDECODE, bad_frame) at exactly the points where
// decode_frames raises DecodeError (fk/codec.py:162-208).
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <vector>

#include "../../include/kvf.h"

namespace kvf {
void set_error(const char* fmt, ...);
}

namespace {

uint32_t rd_u32(const uint8_t* p) {
  uint32_t v;
  memcpy(&v, p, 4);  // little-endian host (x86-64 / aarch64)
  return v;
}

kvf_status decode_error(int32_t* bad, int32_t frame, const char* what) {
  if (bad) *bad = frame;
  kvf::set_error("%s at frame %d", what, frame);
  return KVF_EDECODE;
}

}  // namespace

extern "C" kvf_status kvf_kvfc_scan(const uint8_t* data, int64_t size, kvf_kvfc_info* info,
                                    int64_t* payload_off, int32_t* payload_len,
                                    int64_t* bitmap_off, uint8_t* frame_type,
                                    int32_t cap_frames, int32_t* bad_frame) {
  if (!info || (size > 0 && !data)) {
    kvf::set_error("null argument");
    return KVF_EINVAL;
  }
  if (size < 12) return decode_error(bad_frame, 0, "stream shorter than header");
  const uint32_t n = rd_u32(data), h = rd_u32(data + 4), w = rd_u32(data + 8);
  const int64_t bh = ((int64_t)h + 15) / 16, bw = ((int64_t)w + 15) / 16;
  const int64_t blen = (bh * bw + 7) / 8;
  if (n > 0x7FFFFFFF || h > 0x7FFFFFFF || w > 0x7FFFFFFF || blen > 0x7FFFFFFF) {
    kvf::set_error("stream header out of range");
    return KVF_EUNSUPPORTED;
  }
  info->n_frames = (int32_t)n;
  info->height = (int32_t)h;
  info->width = (int32_t)w;
  info->bitmap_len = (int32_t)blen;
  // A frame takes at least 13 bytes (type + three u32 lengths): a header that
  // claims more frames than the bytes can hold is truncated, and the walk below
  // (without filling) finds the frame decode_frames would raise at.  Callers
  // size their arrays from n only after this check, so a corrupt header cannot
  // make them allocate n-sized arrays.
  const bool fits = 13 * (int64_t)n + 12 <= size;
  if (cap_frames < (int64_t)n && fits) {  // size query: the walk runs on the fill call
    kvf::set_error("arrays hold %d frames, stream has %u", cap_frames, n);
    return KVF_EINVAL;
  }
  const bool fill = fits;
  int64_t pos = 12;
  for (int32_t f = 0; f < (int32_t)n; ++f) {
    if (pos >= size) return decode_error(bad_frame, f, "stream truncated");
    const uint8_t type = data[pos++];
    if (type != 0 && type != 1) return decode_error(bad_frame, f, "bad frame type");
    if (type == 1 && f == 0) return decode_error(bad_frame, f, "inter frame without reference");
    if (fill && frame_type) frame_type[f] = type;
    for (int p = 0; p < 3; ++p) {
      const int64_t k = 3 * (int64_t)f + p;
      if (type == 1) {
        if (pos + blen > size) return decode_error(bad_frame, f, "stream truncated");
        if (fill && bitmap_off) bitmap_off[k] = pos;
        pos += blen;
      } else if (fill && bitmap_off) {
        bitmap_off[k] = -1;
      }
      if (pos + 4 > size) return decode_error(bad_frame, f, "stream truncated");
      const uint32_t plen = rd_u32(data + pos);
      pos += 4;
      if (pos + (int64_t)plen > size) return decode_error(bad_frame, f, "stream truncated");
      if (fill) {
        if (payload_off) payload_off[k] = pos;
        if (payload_len) payload_len[k] = (int32_t)plen;
      }
      pos += plen;
    }
  }
  if (pos != size) return decode_error(bad_frame, (int32_t)n - 1, "trailing bytes");
  return KVF_OK;
}

// Many streams: a header pass (frame_base == NULL: infos only) or the fill pass
// over up to n_threads host threads, stream j's frames at frame_base[j] of the
// flat arrays.  The walk is a pointer chase with one cache miss per plane, so
// streams are spread over threads; one call replaces a Python-level loop of
// two kvf_kvfc_scan calls per stream.  On an error the first failing stream
// (in order) is walked again on the calling thread, so kvf_last_error()
// describes it; *bad_stream / *bad_frame locate it.
extern "C" kvf_status kvf_kvfc_scan_batch(const uint8_t* const* data, const int64_t* size,
                                          int32_t n_streams, kvf_kvfc_info* info,
                                          const int64_t* frame_base, int64_t* payload_off,
                                          int32_t* payload_len, int64_t* bitmap_off,
                                          uint8_t* frame_type, int32_t n_threads,
                                          int32_t* bad_stream, int32_t* bad_frame) {
  if (n_streams < 0 || (n_streams > 0 && (!data || !size || !info))) {
    kvf::set_error("null argument");
    return KVF_EINVAL;
  }
  if (bad_stream) *bad_stream = -1;
  const bool fill = frame_base != nullptr;
  if (fill && (!payload_off || !payload_len || !bitmap_off || !frame_type)) {
    kvf::set_error("null output array");
    return KVF_EINVAL;
  }
  std::vector<kvf_status> st(n_streams, KVF_OK);
  auto walk = [&](int32_t j, int32_t* bad) -> kvf_status {
    if (!fill) {  // header: a size query (KVF_EINVAL with info filled is success)
      const kvf_status s = kvf_kvfc_scan(data[j], size[j], &info[j], nullptr, nullptr, nullptr,
                                         nullptr, 0, bad);
      return s == KVF_EINVAL && size[j] >= 12 ? KVF_OK : s;
    }
    const int64_t b = frame_base[j];
    return kvf_kvfc_scan(data[j], size[j], &info[j], payload_off + 3 * b, payload_len + 3 * b,
                         bitmap_off + 3 * b, frame_type + b, (int32_t)info[j].n_frames, bad);
  };
  const int32_t nt = std::max(1, std::min<int32_t>(fill ? n_threads : 1, n_streams));
  std::atomic<int32_t> next(0);
  auto worker = [&]() {
    for (int32_t j; (j = next.fetch_add(1)) < n_streams;) {
      int32_t bad = 0;
      st[j] = walk(j, &bad);
    }
  };
  if (nt == 1) {
    worker();
  } else {
    std::vector<std::thread> pool;
    try {
      for (int32_t t = 1; t < nt; ++t) pool.emplace_back(worker);
    } catch (...) {  // no threads available: the calling thread walks the rest
    }
    worker();
    for (auto& t : pool) t.join();
  }
  for (int32_t j = 0; j < n_streams; ++j) {
    if (st[j] == KVF_OK) continue;
    int32_t bad = 0;
    const kvf_status s = walk(j, &bad);  // again on this thread: its error message
    if (bad_stream) *bad_stream = j;
    if (bad_frame) *bad_frame = bad;
    return s;
  }
  return KVF_OK;
}
