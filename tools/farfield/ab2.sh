# far-field variants on configs 3 and 5 (development aid): ab2.sh variant...
cd ${GRAFT_REPO_ROOT:-.}
for v in "$@"; do
  if [ $v = default ]; then unset GWN_B200_LIB; else export GWN_B200_LIB=$PWD/build/variants/libgwn_b200_$v.so; fi
  echo "== $v"; timeout 600 python tools/farfield/check.py 3 4194304 gpurun_out/f3_$v.npz; timeout 600 python tools/farfield/check.py 5 1048576 gpurun_out/f5_$v.npz
done
