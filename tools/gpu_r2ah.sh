echo "== current"; python tools/dbg_fuse_edges.py
cp paper_2407_18015_b200/libcritprob_b200.so /tmp/keep.so; cp ab/old.so paper_2407_18015_b200/libcritprob_b200.so
echo "== old"; python tools/dbg_fuse_edges.py
cp /tmp/keep.so paper_2407_18015_b200/libcritprob_b200.so
