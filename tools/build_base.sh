# build the committed (HEAD or $1) sources as build/variants/libamsq_base.so for A/B timing
set -e
cd "$(dirname "$0")/.."
REV=${1:-HEAD}
rm -rf /tmp/amsq_base && git worktree add -f /tmp/amsq_base $REV > /dev/null 2>&1
NCCL_INC=$(python -c "import nvidia.nccl as n,os;print(os.path.join(list(n.__path__)[0],'include'))")
NCCL_LIB=$(python -c "import nvidia.nccl as n,os;print(os.path.join(list(n.__path__)[0],'lib'))")
mkdir -p build/variants
objs=""
for src in /tmp/amsq_base/paper_2510_16045_b200/csrc/*.cu /tmp/amsq_base/paper_2510_16045_b200/csrc/*.cpp; do
  o=build/variants/base_$(basename $src).o
  x=""; case $src in *.cpp) x="-x cu";; esac
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -lineinfo -Xcompiler -fPIC -I /tmp/amsq_base/include -I /tmp/amsq_base/paper_2510_16045_b200/csrc -I $NCCL_INC --expt-relaxed-constexpr $x -c $src -o $o &
  objs="$objs $o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/libamsq_base.so $objs -L $NCCL_LIB -l:libnccl.so.2 -Xlinker -rpath=$NCCL_LIB -lcudart
git worktree remove --force /tmp/amsq_base
echo built build/variants/libamsq_base.so from $REV
