"""Generate tests/golden/presets.json from the REFERENCE implementation:
the layer lists of its three network presets (``builtin_network``,
layers.py:100-106, over presets/*.cfg) and its four parameter sweeps
(``sweep``, layers.py:114-135), plus the Eq. 1 scratch of every sweep
geometry as the reference's own meter counts it (im2col lowered matrix vs
the SMM slice buffer, test_acceptance.py:127-153).  Build container only:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_presets.py
"""
import json
from pathlib import Path

from smmconv import random_tensor, repack_weights, smm_conv_single
from smmconv.im2col import im2col_pack
from smmconv.layers import NETWORK_NAMES, SWEEP_KINDS, builtin_network, sweep
from smmconv.workspace import metered

OUT = Path(__file__).resolve().parent / "presets.json"


def geom(g):
    return [g.in_channels, g.out_channels, g.in_h, g.in_w, g.k_h, g.k_w,
            g.stride_h, g.stride_w, g.pad_h, g.pad_w]


def main():
    data = {"networks": {n: [[s.name, geom(s.geometry)] for s in builtin_network(n)]
                         for n in NETWORK_NAMES},
            "sweeps": {}}
    for kind in SWEEP_KINDS:
        rows = []
        for s in sweep(kind):
            g = s.geometry
            inp = random_tensor(g.input_shape, 17)
            with metered() as m_pack:
                im2col_pack(inp, g)
            w_smm = repack_weights(random_tensor(g.weights_shape, 18), g)
            with metered() as m_smm:
                smm_conv_single(inp, w_smm, g)
            rows.append([s.name, geom(g), m_pack.total_alloc_elements(),
                         m_smm.total_alloc_elements()])
        data["sweeps"][kind] = rows
    OUT.write_text(json.dumps(data, indent=0))
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
