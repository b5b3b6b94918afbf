for e in cr2 ref; do SEELE_LIB=tools/_libs/prof.so python tools/raster_counts.py --engine $e 2>&1 | tail -3; done
