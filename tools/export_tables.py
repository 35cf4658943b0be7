"""Re-serialise the reference's shipped i_max=256 tables into the binary ZIGT form.

Run once in the build container (the reference tree is not present on the GPU
box):  python tools/export_tables.py [/root/reference/pkg/src/zigfast/data]

Input: the reference's JSON fixtures (`zigfast/data/{exponential,halfnormal}_256.json`,
checked against their CRC32 by `tables.from_json_bytes`).  Output:
`paper_1403_6870_b200/data/<kind>_256.zigt` — the same float64 bits in the
reference's own binary container (`zigfast/tableio.py:97-143`).
"""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_1403_6870_b200 import tables as T  # noqa: E402

src = pathlib.Path(sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src/zigfast/data")
dst = pathlib.Path(__file__).resolve().parents[1] / "paper_1403_6870_b200" / "data"
dst.mkdir(exist_ok=True)
for kind in (T.EXPONENTIAL, T.HALF_NORMAL):
    tab = T.from_json_bytes((src / f"{kind}_256.json").read_bytes())
    blob = T.to_binary(tab)
    assert T.from_binary(blob) == tab
    (dst / f"{kind}_256.zigt").write_bytes(blob)
    print(kind, "l_max", tab.l_max, "X[1]", tab.x[1], "eps", tab.epsilon_max, len(blob), "bytes")
