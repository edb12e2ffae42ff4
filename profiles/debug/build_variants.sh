# build profiling variants of libsmx.so: profiles/debug/var/libsmx_<NAME>.so with -D<FLAGS>
# usage: build_variants.sh NAME:FLAG[,FLAG] ...
mkdir -p profiles/debug/var
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  defs=""; for f in ${flags//,/ }; do defs="$defs -D$f"; done
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -shared -Iinclude $defs -o profiles/debug/var/libsmx_$name.so paper_2006_11972_b200/csrc/smx.cu &
done
wait
ls -la profiles/debug/var
