# Build libomcg.so of git revision <rev> into ab_libs/<name>/ (A/B against the
# working tree): bash scripts/ab_build_rev.sh <name> <rev> [-DFLAG=value ...]
set -e
name=$1; rev=$2; shift 2
root=$(pwd)
tmp=$(mktemp -d)
git archive "$rev" paper_2402_09222_b200/csrc include | tar -x -C "$tmp"
mkdir -p "$root/ab_libs/$name"
make -s -C "$tmp/paper_2402_09222_b200/csrc" PKG="$root/ab_libs/$name" KFLAGS="$*" "$root/ab_libs/$name/libomcg.so"
rm -rf "$tmp"
