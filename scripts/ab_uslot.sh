#!/usr/bin/env bash
# A/B of the uniform-slot SpMV geometry (slices per iteration, CTAs/SM):
# pell_probe (7-pt 128^3, 27-pt 256^3) and the bench solve's SpMV phase.
bash scripts/ab_ppat.sh "" "-DUSLOT_U=2" "-DUSLOT_U=2 -DUSLOT_MIN_BLOCKS=3" "-DUSLOT_MIN_BLOCKS=6" ""
