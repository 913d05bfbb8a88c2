set -e
cd "$(dirname "$0")"
R=../../paper_2305_10611_b200
for f in backend runtime zoo capi jit pool; do g++ -O2 -g -pg -std=c++20 -fPIC -ffp-contract=off -I../../include -I$R/csrc -I$R/build/gen -I/usr/local/cuda/include -c $R/csrc/$f.cpp -o $f.o & done; wait
g++ -O2 -g -pg -std=c++20 -I../../include drv.cpp backend.o runtime.o zoo.o capi.o jit.o pool.o $R/build/obj/kernels_vm.cu.o $R/build/obj/kernels_tc.cu.o $R/build/obj/kernels_mv.cu.o -L/usr/local/cuda/lib64 -lcudart_static -lpthread -ldl -lrt -o drv
