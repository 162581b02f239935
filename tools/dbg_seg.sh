cd $GRAFT_REPO_ROOT
for name in small_box c1; do for k in 2 4 5 6; do for g in 1; do
  SPFD_DEBUG=1 timeout 120 python -X faulthandler tools/dbg_seg.py $k $g $name > /tmp/o.txt 2>&1; echo "rc=$? k=$k g=$g $name"; grep -E "^[0-9]|Error|error|spfd|File.*paper" /tmp/o.txt | head -5
done; done; done
