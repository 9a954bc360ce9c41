# SASS of k_scan_refine_ed<0,0> from a built library (blank lines dropped) -> stdout
so=${1:-paper_2110_07519_b200/libmessi.so}
cuobjdump -sass "$so" > /tmp/_all.sass
L=$(grep -n 'Function : _ZN5messi16k_scan_refine_edILb0ELb0' /tmp/_all.sass | cut -d: -f1)
awk -v L=$L 'NR>L && /Function :/ {exit} NR>=L' /tmp/_all.sass | grep -v '^\s*$' | grep -v '^\s*/\* [0-9a-f]* \*/\s*$'
