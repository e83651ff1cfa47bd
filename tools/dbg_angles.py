"""Dev tool: angle-split p2p reduction at a given size (debugging)."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_2505_13955_b200.distributed import AngleSplitReconstructor
from paper_2505_13955_b200.engine import phantom_raw
from paper_2505_13955_b200.geometry import AcquisitionParams, VolumeDims
n, n_proj, rows = (int(x) for x in sys.argv[1:4])
local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local); dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
p = AcquisitionParams(n_proj=n_proj, n_rows=rows, n_chan=n, pixel_pitch=12.0)
d = VolumeDims(n, n, rows, voxel_pitch=12.0)
z = AngleSplitReconstructor(p, d, i0=1e5, reduce="p2p", device=dev)
print(dist.get_rank(), "ptrs", [hex(x) for x in z.symm.buffer_ptrs], hex(z.slab.data_ptr()), z.slab.numel() * 4, flush=True)
if os.environ.get("DBG_LOCAL"):
    z._dst = (ctypes.c_void_p * z.world)(*([z.slab.data_ptr()] * z.world))
if os.environ.get("DBG_PLAIN"):  # ordinary allocation instead of symmetric memory
    z.slab = torch.empty_like(z.slab)
    z._dst = (ctypes.c_void_p * z.world)(*([z.slab.data_ptr()] * z.world))
if os.environ.get("DBG_NOFIN"):
    import paper_2505_13955_b200.distributed as D
    class L:
        def __getattr__(self, k):
            f = getattr(D.lib(), k)
            return (lambda *a: 0) if k == "tf_bp_finalize" else f
    D.lib = lambda: L()
chunk = torch.empty(z.chunk_shape(), device=dev)
phantom_raw(p, d, chunk, a0=z.a0, a1=z.a1)
for i in range(3):
    z.run(chunk)
    torch.cuda.synchronize()
    print(dist.get_rank(), "run", i, flush=True)
    torch.cuda.synchronize()
    print(dist.get_rank(), "step", i, "ok", flush=True)
dist.barrier()
dist.destroy_process_group()
