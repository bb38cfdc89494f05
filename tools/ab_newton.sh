# A/B of library variants in build/variants (development aid): ab_newton.sh v1 v2 ...
cd ${GRAFT_REPO_ROOT:-.}
for v in "$@"; do
  if [ $v = default ]; then unset GWN_B200_LIB; else export GWN_B200_LIB=$PWD/build/variants/libgwn_b200_$v.so; fi
  echo "== $v"; timeout 300 bash tools/quick_bench.sh 3
done
