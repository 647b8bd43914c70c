for d in 4 32; do MGK_PBR_PROFILE=1 timeout 600 python -c "
import sys, time; sys.path.insert(0, '.')
from paper_1910_06310_b200 import native, synth
ds = synth.config4(count=2, degrees=($d,))
ctx = native.Context(0); ctx.upload(native.PackedDataset(ds)); ctx.set_kernels(None, None)
t = time.time(); ctx.reorder_pbr(0, False); print('deg $d', [g.node_count for g in ds], 'PBR', round(time.time() - t, 2), 's')
" 2>&1 | tail -2; done
