"""Run one multi-process peer-transport case by hand (tests/_peer_worker.py),
printing every rank's phase timestamps.   python tools/peer_group.py CASE PROCS"""
import os, subprocess, sys, tempfile, uuid
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
case, procs = sys.argv[1], int(sys.argv[2])
d = tempfile.mkdtemp()
g = f"/eb_m{uuid.uuid4().hex[:12]}"
ps = [subprocess.Popen([sys.executable, os.path.join(HERE, "tests", "_peer_worker.py"), case,
                        str(procs), str(r), g, d, "2"]) for r in range(procs)]
print([p.wait() for p in ps])
