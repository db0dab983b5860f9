"""Generate the golden fixtures in tests/golden/ from the reference's OWN
sources (oracle/_ref/libocw_ref.so, built by oracle/build_ref.sh from
/root/reference/proj/src).  Inputs are regenerated from seeds with the
reference's own fixture generator (matrix.cpp:57-62 random_gaussian), so only
outputs are stored.

    OCW_SHIM_NO_BLAS=1 python tests/golden/make_golden.py

(fixed-order fp64 loops in the shim -> bit-identical on any x86-64 host).
"""
import hashlib
import os
import sys
from pathlib import Path

os.environ.setdefault("OCW_SHIM_NO_BLAS", "1")
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from oracle import ocw_oracle as orc  # noqa: E402
from oracle import ref  # noqa: E402

OUT = Path(__file__).resolve().parent

# name: (n, m, t, seed_w, sd_w, seed_x, bf16, bits, scheme, gran, group, actorder, block)
CASES = {
    # BASELINE config 1 (runs on the CPU reference): 512x512, 4096 bf16 tokens,
    # 4-bit asymmetric g128, block 128, no act-order
    "c1_512x512_w4g128": (512, 512, 4096, 0x5EED0010, 0.02, 0x5EED1010, 1, 4, 1, 2, 128, 0, 128),
    "small_sym3_channel_act": (64, 96, 256, 11, 0.02, 12, 1, 3, 0, 1, 0, 1, 32),
    "small_asym2_g32_act": (96, 64, 512, 13, 0.02, 14, 1, 2, 1, 2, 32, 1, 16),
    "small_asym4_tensor": (48, 40, 128, 15, 1.0, 16, 0, 4, 1, 0, 0, 0, 32),
    "small_asym8_g16_block1": (32, 48, 96, 17, 0.05, 18, 1, 8, 1, 2, 16, 1, 1),
}


def main():
    for name, (n, m, t, sw, sdw, sx, bf, bits, scheme, gran, group, act, block) in CASES.items():
        w = ref.random_gaussian(n, m, sw, sdw)
        x = ref.random_gaussian(t, n, sx)
        if bf:
            x = orc.bf16_round(x)
        gram, cross = np.zeros((n, n)), np.zeros((n, n))
        ref.accumulate_stats(gram, cross, x, x)
        h = gram.astype(np.float32)
        codes, s, z = ref.gptq_quantize(w, h, bits, scheme, gran, group, bool(act), 0.01, block)
        cfg = orc.QuantConfig(bits, orc.Scheme(scheme), orc.Granularity(gran), group)
        grids = orc.Grids(s, z, orc.scheme_qmin(bits, orc.Scheme(scheme)),
                          orc.scheme_qmax(bits, orc.Scheme(scheme)))
        payload = np.frombuffer(orc.pack_uniform(codes, grids, cfg), np.uint8)
        w_hat = ref.dequantize(codes, s, z, bits, scheme, gran, group)
        obj = ref.activation_objective(w, w_hat, h)
        obj0 = ref.activation_objective(w, np.zeros_like(w), h)
        hinv, u, damp = ref.gptq_factor(h, bool(act), 0.01)
        np.savez_compressed(
            OUT / f"{name}.npz", kind="gptq", n=n, m=m, t=t, seed_w=sw, sd_w=sdw, seed_x=sx, bf16=bf,
            cfg=np.array([bits, scheme, gran, group, act, block]),
            h_sha256=hashlib.sha256(h.tobytes()).hexdigest(),
            h_diag=np.diagonal(h).copy(), order=ref.gptq_order(h, bool(act)),
            u_diag=np.diagonal(u).copy(), u_row0=u[0].copy(), hinv_diag=np.diagonal(hinv).copy(),
            damp=damp, codes=codes if n * m <= 16384 else np.zeros(0, np.int16), payload=payload,
            scales=s, zeros=z, rel_err=np.sqrt(obj / obj0))
        print(name, payload.size, "bytes payload, rel_err", np.sqrt(obj / obj0))


if __name__ == "__main__":
    main()
