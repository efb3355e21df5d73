import os, sys
os.environ["DEFORMTRACK_B200_LIB"] = "/root/repo/tools/libdt_debug.so"
sys.path.insert(0, "/root/repo")
exec(open("/root/repo/tools/dbg_wr2.py").read().split("print(\"dvalid all\"")[0])
