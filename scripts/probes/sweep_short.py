import json
import sys

for line in sys.stdin:
    d = json.loads(line)
    if "qr_us" in d:
        print(f"N {d['N']:>10} M {d['M']:>2} qr_us {d['qr_us']:9.1f} ex_us {d['extrap_us']:8.1f}")
