"""Probe the box's video engines for SURVEY.md section 8f row 4 (NVDEC variant).

* NVDEC: dlopen libnvcuvid (driver-provided; the image ships no Video Codec SDK
  headers, so CUVIDDECODECAPS is declared here from the SDK's cuviddec.h layout)
  and query cuvidGetDecoderCaps for HEVC 4:4:4 / 4:2:0 8-bit and H.264 4:2:0:
  supported?, number of NVDEC engines, min/max frame size.
* NVENC: NVML nvmlDeviceGetEncoderCapacity (0 = no encoder capacity).

    python tools/probe_nvdec.py > gpurun_out/probe_nvdec.json
"""

from __future__ import annotations

import ctypes
import json

import torch


class CUVIDDECODECAPS(ctypes.Structure):
    _fields_ = [
        ("eCodecType", ctypes.c_int),          # cudaVideoCodec (IN)
        ("eChromaFormat", ctypes.c_int),       # cudaVideoChromaFormat (IN)
        ("nBitDepthMinus8", ctypes.c_uint),    # IN
        ("reserved1", ctypes.c_uint * 3),
        ("bIsSupported", ctypes.c_ubyte),      # OUT
        ("nNumNVDECs", ctypes.c_ubyte),
        ("nOutputFormatMask", ctypes.c_ushort),
        ("nMaxWidth", ctypes.c_uint),
        ("nMaxHeight", ctypes.c_uint),
        ("nMaxMBCount", ctypes.c_uint),
        ("nMinWidth", ctypes.c_ushort),
        ("nMinHeight", ctypes.c_ushort),
        ("bIsHistogramSupported", ctypes.c_ubyte),
        ("nCounterBitDepth", ctypes.c_ubyte),
        ("nMaxHistogramBins", ctypes.c_ushort),
        ("reserved3", ctypes.c_uint * 10),
    ]


CODECS = {"H264": 4, "HEVC": 8, "AV1": 11}
CHROMA = {"420": 1, "444": 3}


def nvdec():
    out = {}
    try:
        lib = ctypes.CDLL("libnvcuvid.so.1")
    except OSError as e:
        return {"libnvcuvid": f"not loadable: {e}"}
    torch.zeros(1, device="cuda")  # the primary context is current on this thread
    for name, codec, chroma in (("HEVC_444_8bit", "HEVC", "444"), ("HEVC_420_8bit", "HEVC", "420"),
                                ("H264_420_8bit", "H264", "420"), ("AV1_444_8bit", "AV1", "444")):
        caps = CUVIDDECODECAPS()
        caps.eCodecType = CODECS[codec]
        caps.eChromaFormat = CHROMA[chroma]
        caps.nBitDepthMinus8 = 0
        rc = lib.cuvidGetDecoderCaps(ctypes.byref(caps))
        out[name] = {"rc": rc, "supported": bool(caps.bIsSupported), "nvdecs": caps.nNumNVDECs,
                     "min_wh": [caps.nMinWidth, caps.nMinHeight],
                     "max_wh": [caps.nMaxWidth, caps.nMaxHeight],
                     "output_format_mask": caps.nOutputFormatMask}
    return out


def nvenc():
    try:
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(0)
        res = {"name": nv.nvmlDeviceGetName(h)}
        for q, label in ((0, "H264"), (1, "HEVC"), (2, "AV1")):
            try:
                res[f"encoder_capacity_{label}"] = nv.nvmlDeviceGetEncoderCapacity(h, q)
            except Exception as e:  # noqa: BLE001
                res[f"encoder_capacity_{label}"] = f"n/a ({type(e).__name__})"
        return res
    except Exception as e:  # noqa: BLE001
        return {"nvml": f"unavailable: {e}"}


if __name__ == "__main__":
    print(json.dumps({"nvdec": nvdec(), "nvenc": nvenc()}, indent=1))
