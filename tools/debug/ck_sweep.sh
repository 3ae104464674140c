python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
QF_CKPT=0 python tools/debug/ck_e2e2.py
python tools/debug/ck_e2e2.py
QF_CKPT_PAD=4096 python tools/debug/ck_e2e2.py
QF_CKPT_PAD=1060864 python tools/debug/ck_e2e2.py
