python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
python tools/debug/ck_var.py
QF_CKPT_NOMEM=1 python tools/debug/ck_var.py
QF_CKPT_CACHE=1 python tools/debug/ck_var.py
QF_CKPT_CACHE=1 QF_CKPT_NOMEM=1 python tools/debug/ck_var.py
QF_CKPT=0 python tools/debug/ck_var.py
python tools/debug/ck_var.py
