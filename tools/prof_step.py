"""One warm cfg2 step (3 subrates: sense + decode) and one cfg4 IDA batch, for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2001_09632_b200 as p  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
imgs = p.synth_images(p.SynthSpec(512, 512, 20, 5.0, 2), 0, 1024)
p.Context.get().set_pipeline_streams(int(os.environ.get("PROF_STREAMS", "1")))  # 1: one launch = 1024 images
if which in ("all", "cfg2"):
    for rep in range(2):
        for num, den in ((1, 10), (3, 10), (1, 2)):
            b = p.sense_batch(imgs, p.SensingConfig(16, num, den, p.Algorithm.DD))
            p.decode_batch(b)
if which in ("all", "fused"):
    for rep in range(2):
        for num, den in ((1, 10), (3, 10), (1, 2)):
            p.sense_decode_batch(imgs, p.SensingConfig(16, num, den, p.Algorithm.DD))
if which in ("all", "ida"):
    b = p.sense_batch(imgs[:64], p.SensingConfig(16, 3, 10, p.Algorithm.BBV))
    for rep in range(2):
        p.ida_batch(b, p.ReconConfig(p.ReconMethod.Ida, iterations=10), trace=False, check=False)
if which in ("all", "den"):
    import ctypes as C
    from paper_2001_09632_b200 import _lib
    f = imgs[:64].float().contiguous()
    out = torch.empty_like(f)
    sig = (C.c_double * 64)(*([7.0] * 64))
    for rep in range(3):
        rc = _lib.load().abcs_denoise_dct_batch(p.Context.get().handle, f.data_ptr(), 512, 512, 512 * 512, 64, sig,
                                                1.0, 8, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
        assert rc == 0, rc
torch.cuda.synchronize()
print("ok")
