SKIP=${SKIP:-30} COUNT=${COUNT:-6} bash tools/gpu/prof_full.sh bin2 'k_bin'
bash tools/gpu/ab.sh base minb7 minb10 minb12
