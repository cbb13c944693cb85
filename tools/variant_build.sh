# dev: build paper_2411_17651_b200/libpsg_<name>.so with extra -D flags on psg_sim.cu
#   bash tools/variant_build.sh fill4 -DPSG_FILL_B=4
set -e
R=$(cd "$(dirname "$0")/.." && pwd); C=$R/paper_2411_17651_b200/csrc; name=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 \
  -Xcompiler -fPIC -I$R/include -I$C "$@" -c $C/psg_sim.cu -o /tmp/psg_sim_$name.o
case " $* " in
  *PSG_PHASE_PROFILE*) objs=$(ls $C/build/prof_*.o $C/build/host_*.o | grep -v '/prof_psg_sim.o$') ;;
  *) objs=$(ls $C/build/*.o | grep -v -e '/psg_sim.o$' -e '/prof_') ;;
esac
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/paper_2411_17651_b200/libpsg_$name.so \
  /tmp/psg_sim_$name.o $objs -lcudart_static -lrt -lpthread -ldl
