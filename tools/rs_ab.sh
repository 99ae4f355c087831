M="tests/test_multi_device.py::test_multi_matches_single_and_reference[stokeslet_d0-2]"
mapfile -t IDS < tools/ids.txt
for k in 4 5 6 7; do echo "id$k+slab"; python -m pytest -m gpu -x -q "${IDS[@]:$k:1}" "${IDS[@]:8:12}" "$M" 2>&1 | tail -1; done
echo "4-7"; python -m pytest -m gpu -x -q "${IDS[@]:4:4}" "$M" 2>&1 | tail -1
