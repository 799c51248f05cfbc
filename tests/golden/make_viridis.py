"""Vendors the canonical 256-entry viridis colormap (8-bit RGB) as data for
the hit-count heatmap ("viridis colormap represents 0 to 20
times"). Source: OpenCV's COLORMAP_VIRIDIS lookup table, read back by
mapping the ramp 0..255 (the image has no matplotlib). Run once:

    python tests/golden/make_viridis.py
"""
import json
import os

import cv2
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ramp = np.arange(256, dtype=np.uint8).reshape(1, 256)
rgb = cv2.applyColorMap(ramp, cv2.COLORMAP_VIRIDIS)[0][:, ::-1]  # BGR -> RGB
out = os.path.join(ROOT, "paper_2305_07238_b200", "data", "viridis_u8.json")
with open(out, "w") as f:
    json.dump({"source": "OpenCV COLORMAP_VIRIDIS (canonical matplotlib viridis, 8-bit)",
               "rgb": rgb.astype(int).tolist()}, f)
print(out, rgb[0].tolist(), rgb[128].tolist(), rgb[255].tolist())
