"""Which nvJPEG backend opens on this GPU, and why the hardware one does not."""
import io, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2512_17574_b200 as fc
from PIL import Image
for b in ("hardware", "cuda", "auto"):
    try:
        d = fc.JpegDecoder(b)
        print(b, "->", d.backend, d.hardware_error)
        buf = io.BytesIO(); Image.fromarray(np.zeros((64, 64, 3), np.uint8)).save(buf, "JPEG", subsampling=2)
        y, u, v = d.decode(buf.getvalue()); import torch; torch.cuda.synchronize(); print("  decode ok", y.shape)
    except Exception as e:
        print(b, "failed:", e)
