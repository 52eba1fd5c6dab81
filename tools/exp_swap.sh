#!/bin/bash
# run a command with the experiment build of libspgemm swapped in (timing experiments only)
cp paper_1804_01698_b200/libspgemm.so /tmp/libspgemm_keep.so
cp paper_1804_01698_b200/libspgemm_exp.so paper_1804_01698_b200/libspgemm.so
touch paper_1804_01698_b200/libspgemm.so
"$@"
rc=$?
cp /tmp/libspgemm_keep.so paper_1804_01698_b200/libspgemm.so
exit $rc
