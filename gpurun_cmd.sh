python -m pytest tests/test_dict_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
bash scripts/ab_probe.sh "-DPELL_CTAB=0" "" "-DPELL_MIN_BLOCKS=4" "-DPELL_MIN_BLOCKS=6"
bash scripts/ab_quick.sh "-DPELL_CTAB=0" "" "-DPELL_MIN_BLOCKS=4"
