"""Random 32-B sector gather throughput vs buffer size (roofline denominators).
Prints one JSON line: {bytes: GB/s}."""
import json
import sys

sys.path.insert(0, ".")
import paper_1904_12754_b200 as P  # noqa: E402

out = {}
for mb in (16, 64, 128, 256, 512, 1024, 2048, 4096, 8192):
    out[f"{mb}MB"] = round(P.bench_gather(0, mb << 20, 64, 5), 1)
print(json.dumps(out))
