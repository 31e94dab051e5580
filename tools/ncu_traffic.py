"""DRAM bytes (read + write) per launch of the first captured kernel in each
`full_<layer>.ncu-rep` -> JSON {layer: bytes} (bench.py's roofline.traffic).
Usage: python tools/ncu_traffic.py out.json rep [rep...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import raw  # noqa: E402


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
             "GB": 1e9}.get(unit, 1)
    return float(v.replace(",", "")) * scale


def main():
    out = {}
    for rep in sys.argv[2:]:
        recs, units = raw(rep)
        if not recs:
            continue
        r = recs[-1]  # the conv kernel (last capture of the rep)
        b = sum(to_bytes(r[k], units.get(k, "byte")) for k in ("dram__bytes_read.sum",
                                                                 "dram__bytes_write.sum"))
        layer = os.path.basename(rep)[len("full_"):-len(".ncu-rep")]
        out[layer] = int(b)
    with open(sys.argv[1], "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
