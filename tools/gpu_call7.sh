for a in "5 0 4 2" "6 0 4 2" "7 0 4 2" "6 0 1 2" "7 0 1 2"; do timeout 30 ./tools/sp_probe5 $a; done
