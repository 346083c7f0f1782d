"""GPU tier: the decode kernel's records (upy_decode_kernel: the TMA-pipelined
warp path for 3.8-3.10, the shared-memory start-chain walk + warp decode for
3.11) against the reference-order scalar decoder (decode_scalar, the restatement
of decode_instructions, disasm.py:71-172) for every object of every golden set:
status, error attributes, and each record of valid objects field by field."""
import numpy as np
import pytest

from conftest import golden_cases
from helpers import inputs

pytestmark = pytest.mark.gpu


def _device_decode(ar):
    from paper_2403_13839_b200.api import DeviceArena
    from paper_2403_13839_b200.arena import DECODED_DTYPE, INS_DTYPE

    da = DeviceArena(ar)
    da.upload()
    da.run(mode="decode")
    import torch

    torch.cuda.synchronize()
    units = ar.total_code_units + 1
    dec_off = (units * 12 + 255) & ~255
    ws = da.ws.cpu().numpy()
    ins = ws[:units * 12].view(INS_DTYPE)
    dec = ws[dec_off:dec_off + 24 * ar.n_objs].view(DECODED_DTYPE)
    return ins, dec


@pytest.mark.parametrize("gset", ["c1", "c2", "c3", "c4", "snippets", "fuzz", "mutant"])
def test_decode_kernel_matches_scalar_decoder(gset):
    from paper_2403_13839_b200 import arena, hostcheck

    recs = golden_cases([gset])
    ar = arena.pack(inputs(recs))
    ins_d, dec_d = _device_decode(ar)
    ins_h, dec_h = hostcheck.decode(ar)
    objs = ar.section("objs")
    bad = []
    for o in range(ar.n_objs):
        # n_instrs is informational once a decode error is reported (the scalar
        # decoder leaves the count reached, the warp path 0): compare it for OK only
        want = tuple(dec_h[o]) if dec_h[o]["status"] == 0 else (dec_h[o]["status"], dec_h[o]["aux0"], dec_h[o]["aux1"])
        got = tuple(dec_d[o]) if dec_h[o]["status"] == 0 else (dec_d[o]["status"], dec_d[o]["aux0"], dec_d[o]["aux1"])
        if got != want:
            bad.append((o, int(objs[o]["minor"]), tuple(dec_d[o]), tuple(dec_h[o])))
            continue
        if dec_h[o]["status"] == 0:
            base = int(objs[o]["code_off"]) >> 1
            n = int(dec_h[o]["n_instrs"])
            if not np.array_equal(ins_d[base:base + n], ins_h[base:base + n]):
                k = int(np.nonzero(ins_d[base:base + n] != ins_h[base:base + n])[0][0])
                bad.append((o, int(objs[o]["minor"]), "record", k, ins_d[base + k], ins_h[base + k]))
    assert not bad, bad[:5]
