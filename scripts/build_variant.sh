# usage: bash scripts/build_variant.sh NAME "-DFLAG=.." -- builds abtest/librbg_NAME.so with extra nvcc flags, then restores the default build
NAME=$1; FLAGS=$2
mkdir -p abtest
touch paper_1806_07884_b200/csrc/rbg_asm.cuh
RBG_NVCC_EXTRA="$FLAGS" python -c "
import sys; sys.path.insert(0,'.')
from paper_1806_07884_b200 import build; build.build_rbg()"
cp paper_1806_07884_b200/librbg.so abtest/librbg_$NAME.so
