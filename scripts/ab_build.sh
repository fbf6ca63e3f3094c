# Build a compile-time variant of libomcg.so into ab_libs/<name>/ (git-ignored,
# travels with gpurun): bash scripts/ab_build.sh <name> [-DFLAG=value ...]
set -e
name=$1; shift
mkdir -p ab_libs/$name
make -s -C paper_2402_09222_b200/csrc OBJ=_obj_ab_$name PKG=../../ab_libs/$name KFLAGS="$*" ../../ab_libs/$name/libomcg.so
