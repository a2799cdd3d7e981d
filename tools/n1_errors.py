"""Record the north-star N1 numbers: tiDAS-vs-DAS global error (metrics.py:105-112)
on the GPU and in the float64 oracle at cfg2 / cfg4 / cfg5 (the computations of
tests/test_gpu_n1_error.py), as one JSON document."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from tests.test_gpu_n1_error import n1_cfg2, n1_cfg4, n1_cfg5  # noqa: E402

res = {}
for name, fn in (("cfg2_full_grid", n1_cfg2), ("cfg4_16_rows", n1_cfg4),
                 ("cfg5_frame0_24_rows", lambda: n1_cfg5(0)), ("cfg5_frame777_24_rows", lambda: n1_cfg5(777))):
    g, r, chk = fn()
    res[name] = {"global_error_gpu": g, "global_error_oracle": r, "agree_3sf": f"{g:.3g}" == f"{r:.3g}", **chk}
    print(json.dumps({name: res[name]}), flush=True)
print(json.dumps(res))
