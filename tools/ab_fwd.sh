bash tools/ncu_r02.sh
