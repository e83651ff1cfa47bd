import sys, os, numpy as np, torch, traceback
sys.path.insert(0, '.')
from paper_2505_13955_b200 import formats
g = np.load('tests/golden/golden_fbp.npz')
open('/tmp/in.sino','wb').write(g['file_sino'].tobytes())
for rows in (16, 256):
    try:
        dims, dt = formats.reconstruct_file('/tmp/in.sino', '/tmp/out.vol', pixel_pitch=1.0, slab_rows=rows)
        print('ok', rows)
    except Exception as e:
        traceback.print_exc()
raw, params = formats.read_sino_pinned('/tmp/in.sino')
print(raw.is_pinned(), raw.shape, raw.dtype, raw.is_contiguous())
