cd $GRAFT_REPO_ROOT
for v in "$@"; do
  echo "== $v"
  KK_LIB=build/var/libkk_$v.so timeout 600 python -m pytest tests -m gpu -q -x -k "cluster or ccl" 2>&1 | tail -1
  KK_LIB=build/var/libkk_$v.so timeout 300 python tools/ccl_time.py
done
