#!/bin/bash
# Tuning builds of the product library with other compile-time constants of the level-0
# assembly (k_assembly.cu: HOT_ASM_T rows per tile, HOT_ASM_CP records per ring slot, HOT_ASM_S
# ring slots, HOT_ASM_MINB = min CTAs per SM).  Each lands in lib/libhotb200_<name>.so and
# is loaded with HOT_LIB_VARIANT=<name>; the default build is untouched.
#   tools/asm_variants.sh build name "-DHOT_ASM_T=2 ..."      (on the CPU box)
#   tools/asm_variants.sh time  name scene                    (on the GPU box)
set -e
cd "$(dirname "$0")/../paper_1911_07913_b200/csrc"
case "$1" in
  build) make -s -j8 OUT=../lib/libhotb200_$2.so OBJDIR=../../build/obj_$2 NVEXTRA="$3" ;;
  time) cd ../..; HOT_LIB_VARIANT=$2 python tools/profile_scene.py ${3:-scenes/cfg2_twisting_bars.json} --steps 4 --warmup 2 | grep -E '"assemble_rows": [0-9.]+,|wall_ms' ;;
esac
