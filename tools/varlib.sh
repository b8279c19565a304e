#!/bin/bash
# variant build for A/B experiments: tools/varlib.sh NAME SRC.cu "NVCC FLAGS"
# recompiles one source with extra flags, links it with the other objects of build/ into
# explib/NAME/librtucker_b200.so (select it with RTB_LIB_PATH=explib/NAME/librtucker_b200.so)
set -e
cd "$(dirname "$0")/.."
NAME=$1; SRC=$2; EXTRA=$3
python -m paper_2107_10654_b200.build > /dev/null
mkdir -p explib/$NAME
B=paper_2107_10654_b200
/usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Iinclude $EXTRA \
  -c $B/csrc/$SRC -o explib/$NAME/${SRC%.cu}.o
OBJS=""
for s in k_small k_ttm k_draw k_gram k_chol k_pcg k_fsketch k_c4 k_eig k_hjsvd toolkit verify engine capi; do o=$B/build/$s.o
  if [ "$(basename $o)" = "${SRC%.cu}.o" ]; then OBJS="$OBJS explib/$NAME/${SRC%.cu}.o"; else OBJS="$OBJS $o"; fi
done
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o explib/$NAME/librtucker_b200.so $OBJS -ldl
echo explib/$NAME/librtucker_b200.so
