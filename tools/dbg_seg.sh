cd $GRAFT_REPO_ROOT
for name in c1 small_box; do for k in 2 4 5; do for g in 0 1; do
  timeout 120 python -X faulthandler tools/dbg_seg.py $k $g $name > /tmp/o.txt 2>&1; echo "rc=$? k=$k g=$g $name"; grep -E "^[0-9]|Error|error|File.*paper" /tmp/o.txt | head -5
done; done; done
