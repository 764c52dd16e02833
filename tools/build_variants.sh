# build experimental K2 variants (consumer-warp counts) as separate libraries under build/variants
set -e
cd "$(dirname "$0")/.."
NCCL_INC=$(python -c "import nvidia.nccl as n,os;print(os.path.join(list(n.__path__)[0],'include'))")
NCCL_LIB=$(python -c "import nvidia.nccl as n,os;print(os.path.join(list(n.__path__)[0],'lib'))")
mkdir -p build/variants
# args: NAME=DEFINES pairs, e.g. w20="-DAMSQ_K2_WARPS=20" mode1="-DAMSQ_K2_MODE=1"
for spec in "$@"; do
  W=${spec%%=*}; DEFS=${spec#*=}
  objs=""
  for src in paper_2510_16045_b200/csrc/*.cu paper_2510_16045_b200/csrc/*.cpp; do
    o=build/variants/$(basename $src).w$W.o
    x=""; case $src in *.cpp) x="-x cu";; esac
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -lineinfo -Xcompiler -fPIC -I include -I paper_2510_16045_b200/csrc -I $NCCL_INC --expt-relaxed-constexpr $DEFS $x -c $src -o $o &
    objs="$objs $o"
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/libamsq_$W.so $objs -L $NCCL_LIB -l:libnccl.so.2 -Xlinker -rpath=$NCCL_LIB -lcudart
done
