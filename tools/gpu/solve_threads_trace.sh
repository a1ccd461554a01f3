cd "$(dirname "$0")/../.."
cp paper_2409_03807_b200/_lib/liblipsub_b200.so /tmp/lib_orig.so
for f in /tmp/lib_orig.so _explibs/t384.so; do
  cp "$f" paper_2409_03807_b200/_lib/liblipsub_b200.so
  echo "== $f"
  echo cold; timeout 120 python tools/solve_trace.py --flush c2 2>&1 | tail -1
  echo warm; timeout 120 python tools/solve_trace.py c2 2>&1 | tail -1
  python - <<'P'
import sys; sys.path.insert(0,'.')
from paper_2409_03807_b200 import configs
pr=configs.build("c2"); s=pr.system(); print(s.solve_kernel_info())
P
done
cp /tmp/lib_orig.so paper_2409_03807_b200/_lib/liblipsub_b200.so
