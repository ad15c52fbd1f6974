import sys; sys.path.insert(0, '/root/repo')
import paper_1307_2982_b200._lib as L
L.LIB_PATH = '/root/repo/tools/probe/dbg/libmihg.so'
exec(open('/root/repo/tools/probe/scan_small.py').read())
