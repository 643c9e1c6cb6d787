# Build libnat variants that differ only in bem.cu compile-time tuning macros:
#   bash scripts/build_variants.sh NAME "-DMACRO=V ..." [NAME "-D..."]...
# Each lands in paper_2506_06190_b200/_variants/libnat_NAME.so (git-ignored; travels with gpurun).
set -e
cd "$(dirname "$0")/.."
[ -n "$NAT_SKIP_MAIN" ] || python -m paper_2506_06190_b200.build > /dev/null
P=paper_2506_06190_b200
INC=$(python -c "import nvidia.nccl as m; print(list(m.__path__)[0])")
mkdir -p $P/_variants
pids=()
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  (
    /usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
      -I $INC/include -gencode arch=compute_100a,code=sm_100a $defs -c $P/csrc/bem.cu -o /tmp/bem_$name.o
    objs=$(ls $P/_build/*.o | grep -v '/bem.o$')
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/_variants/libnat_$name.so \
      /tmp/bem_$name.o $objs -L $INC/lib -l:libnccl.so.2 -Xlinker -rpath,$INC/lib
    echo "built $name ($defs)"
  ) &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
