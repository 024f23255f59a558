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
