# Build the library of a git revision into variants/libmdcuda_TAG.so (A/B timing against it)
# usage: bash scripts/build_ref_variant.sh REV TAG
set -e
REV=${1:-HEAD}; TAG=${2:-head}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
WT=/tmp/md_wt_$TAG
rm -rf "$WT"; git -C "$ROOT" worktree prune
git -C "$ROOT" worktree add -q "$WT" "$REV"
(cd "$WT" && python -c "from paper_1212_2245_b200 import build as B; B.build()")
mkdir -p "$ROOT/variants"; cp "$WT/paper_1212_2245_b200/libmdcuda.so" "$ROOT/variants/libmdcuda_$TAG.so"
git -C "$ROOT" worktree remove --force "$WT"
echo "$ROOT/variants/libmdcuda_$TAG.so"
