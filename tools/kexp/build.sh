# Build the experiment harness once per macro setting: tools/kexp/build.sh NAME [-DFLAG=V ...]
set -e
D=$(cd "$(dirname "$0")" && pwd)
R=$(cd "$D/../.." && pwd)
name=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
  -I "$D/tuning" -I "$R/paper_2512_15595_b200/csrc" -I "$R/include" "$@" -o "$D/kexp_$name" "$D/kexp.cu"
