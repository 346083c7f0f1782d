"""Stack-depth analysis of code objects on the GPU (north-star subsystem 3,
SURVEY Appendix A): `stack_depths(codes)` decodes every object with the decode
kernel, then runs the segmented-scan kernel (csrc/stackscan_kernel.cu) over the
records.  Per object: `(records, info)` -- records is a structured array with one
(depth, flags) per instruction (upy_stackrec, include/upy.h) and info the
upy_stackinfo summary; objects that fail to decode carry the decode status in
info and no records."""
from __future__ import annotations


def stack_depths(codes, device=None):
    import torch

    from .api import DeviceArena
    from .arena import STACKINFO_DTYPE, STACKREC_DTYPE, pack

    codes = list(codes)
    if not codes:
        return []
    ar = pack(codes)
    da = DeviceArena(ar, device=device)
    da.upload()
    da.run(mode="decode")
    stack, info = da.stackscan()
    torch.cuda.synchronize(da.device)
    recs = stack.cpu().numpy().view(STACKREC_DTYPE)
    inf = info.cpu().numpy().view(STACKINFO_DTYPE)
    dec = da.decoded()
    objs, roots = ar.section("objs"), ar.section("roots")
    out = []
    for o in roots:
        o = int(o)
        base = int(objs[o]["code_off"]) >> 1
        n = int(dec[o]["n_instrs"]) if int(dec[o]["status"]) == 0 else 0
        out.append((recs[base:base + n].copy(), inf[o].copy()))
    return out
