# like ab_build.sh, but the flags go to the host-side transport.cu too (NVFLAGS)
set -e
name=$1; shift
mkdir -p ab_libs/$name
make -s -C paper_2402_09222_b200/csrc OBJ=_obj_ab_$name PKG=../../ab_libs/$name KFLAGS="$*" NVFLAGS_EXTRA="$*" ../../ab_libs/$name/libomcg.so
