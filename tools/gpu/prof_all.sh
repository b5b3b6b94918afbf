# ncu --set full of every kernel of one steady-state C3 frame + raster phase counts
SKIP=${SKIP:-44} COUNT=${COUNT:-11} bash tools/gpu/prof_full.sh all 'k_'
for e in cr2 ref; do SEELE_LIB=tools/_libs/prof.so python tools/raster_counts.py --engine $e 2>&1 | tail -3; done
