"""Device codecs vs the reference's cv2 on one band-sized image.

    python tools/codec_bench.py [rows] [cols]

Encode: a smooth+noise uint8 code plane -> PNG and deflate TIFF (device bytes
ready on the host) vs cv2.imencode.  Decode: a 16-bit band written by cv2 as
deflate TIFF (what the reference's save_image writes) -> device planes vs
cv2.imdecode.  Wall clock, best of 3, file I/O excluded on both sides.
"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import cv2  # noqa: E402

from paper_1612_06457_b200 import image_io  # noqa: E402


def best(fn, reps=3):
    out, ts = None, []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return out, min(ts)


rows = int(sys.argv[1]) if len(sys.argv) > 1 else 7216
cols = int(sys.argv[2]) if len(sys.argv) > 2 else 5412
rng = np.random.default_rng(0)
y, x = np.mgrid[0:rows, 0:cols]
smooth = (np.sin(x / 37.0) + np.cos(y / 23.0) + 2) / 4
code8 = np.clip(smooth * 255 + rng.normal(0, 1.0, smooth.shape), 0, 255).astype(np.uint8)
band16 = np.clip(smooth * 4095 + rng.normal(0, 4.0, smooth.shape), 0, 4095).astype(np.uint16)
dev8 = torch.from_numpy(code8).cuda()
res = {"image": f"{rows}x{cols}"}
png, res["png_encode_device_s"] = best(lambda: image_io.encode_png(dev8))
ok, ref_png = cv2.imencode(".png", code8)
_, res["png_encode_cv2_s"] = best(lambda: cv2.imencode(".png", code8))
res["png_bytes_device"], res["png_bytes_cv2"] = len(png), int(ref_png.size)
tif, res["tiff_deflate_encode_device_s"] = best(lambda: image_io.encode_tiff(dev8, "deflate"))
_, res["tiff_deflate_encode_cv2_s"] = best(
    lambda: cv2.imencode(".tif", code8, [cv2.IMWRITE_TIFF_COMPRESSION, 8]))
ok, band_tif = cv2.imencode(".tif", band16, [cv2.IMWRITE_TIFF_COMPRESSION, 8])
data = band_tif.tobytes()
got, res["tiff16_decode_device_s"] = best(lambda: image_io.decode_tiff(data))
_, res["tiff16_decode_cv2_s"] = best(
    lambda: cv2.imdecode(np.frombuffer(data, np.uint8), cv2.IMREAD_UNCHANGED))
res["tiff16_strips"] = len(image_io._tiff_layout(data)["offsets"])
assert np.array_equal(got.cpu().numpy(), band16)
# PNG and LZW TIFF bands as cv2 writes them, one file and a 16-band batch
ok, band_png = cv2.imencode(".png", band16)
pdata = band_png.tobytes()
got, res["png16_decode_device_s"] = best(lambda: image_io.decode_png(pdata))
_, res["png16_decode_cv2_s"] = best(
    lambda: cv2.imdecode(np.frombuffer(pdata, np.uint8), cv2.IMREAD_UNCHANGED))
assert np.array_equal(got.cpu().numpy(), band16)
_, res["png16_decode_device_16_files_s"] = best(lambda: image_io.decode_batch([pdata] * 16), reps=2)
ok, band_lzw = cv2.imencode(".tif", band16, [cv2.IMWRITE_TIFF_COMPRESSION, 5])
ldata = band_lzw.tobytes()
got, res["lzw16_decode_device_s"] = best(lambda: image_io.decode_tiff(ldata))
_, res["lzw16_decode_cv2_s"] = best(
    lambda: cv2.imdecode(np.frombuffer(ldata, np.uint8), cv2.IMREAD_UNCHANGED))
assert np.array_equal(got.cpu().numpy(), band16)
res["lzw16_strips"] = len(image_io._tiff_layout(ldata)["offsets"])
# the 8-bit code plane (compressible: match-heavy streams), as cv2 and as the device write it
c8 = ref_png.tobytes()
got, res["png8_cv2file_decode_device_s"] = best(lambda: image_io.decode_png(c8))
assert np.array_equal(got.cpu().numpy(), code8)
_, res["png8_cv2file_decode_cv2_s"] = best(
    lambda: cv2.imdecode(np.frombuffer(c8, np.uint8), cv2.IMREAD_UNCHANGED))
got, res["png8_devfile_decode_device_s"] = best(lambda: image_io.decode_png(png))
assert np.array_equal(got.cpu().numpy(), code8)
_, res["tiff16_decode_device_16_files_s"] = best(lambda: image_io.decode_batch([data] * 16), reps=2)
_, res["lzw16_decode_device_16_files_s"] = best(lambda: image_io.decode_batch([ldata] * 16), reps=2)
print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in res.items()}))
