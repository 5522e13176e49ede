"""One wavefront-QR launch at k (for ncu): python tools/qr_one.py [k]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import qr_ab  # noqa: E402
k = int(sys.argv[1]) if len(sys.argv) > 1 else 120
l, i, t, q, A, B = qr_ab.run(k, 2, False, 0, reps=1)
print(k, t, q[:5])
