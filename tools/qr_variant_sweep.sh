# time the wavefront QR with each prebuilt libcirr_<variant>.so swapped in (A/B of build-time knobs)
cp paper_2511_01927_b200/libcirr.so /tmp/libcirr_default.so
for f in default paper_2511_01927_b200/libcirr_*.so; do
  if [ "$f" != default ]; then cp "$f" paper_2511_01927_b200/libcirr.so; fi
  echo "variant $f"
  timeout 200 python tools/qr_ab.py 2>&1 | grep -E "k=(120|256) seed=0" | sed 's/window.*wavefront/wavefront/' | cut -c1-110
  cp /tmp/libcirr_default.so paper_2511_01927_b200/libcirr.so
done
