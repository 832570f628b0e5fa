# Builds an experimental library variant for A/B timing:
#   tools/variant.sh NAME -DFLAG ...  ->  paper_2312_06902_b200/_lib/libperseus_b200_NAME.so
# (select it with PB_LIB_VARIANT=_NAME).  The default build is untouched.
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
make -s -C "$R/paper_2312_06902_b200/csrc" >/dev/null
/usr/local/cuda/bin/nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -Xcompiler -fPIC \
  -I"$R/include" -I"$R/paper_2312_06902_b200/csrc" "$@" -c "$R/paper_2312_06902_b200/csrc/pb_kernels.cu" -o /tmp/pbk_$name.o
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -cudart static /tmp/pbk_$name.o \
  "$R/paper_2312_06902_b200/_build/pb_host.o" -o "$R/paper_2312_06902_b200/_lib/libperseus_b200_$name.so" -lpthread
echo "built _lib/libperseus_b200_$name.so"
