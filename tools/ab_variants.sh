set -x
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in "$@"; do
  echo "== $v"
  KK_LIB=build/var/libkk_$v.so KK_ONLY_PLANAR=1 timeout 300 python tools/planar_rate.py 65536 16384 4096
done
done
