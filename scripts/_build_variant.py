"""scratch: build libgcb200 variants with a modified h2mv.cu into _scratch/"""
import subprocess, os, shutil, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import build_native as b


def build(name, src, extra=()):
    d = '_scratch/src_' + name + '/csrc'
    shutil.rmtree('_scratch/src_' + name, ignore_errors=True)
    shutil.copytree('paper_1810_08429_b200/csrc', d)
    os.symlink(os.path.abspath('include'), '_scratch/include') if not os.path.exists('_scratch/include') else None
    open(d + '/h2mv.cu', 'w').write(src)
    srcs = sorted(os.path.join(d, f) for f in os.listdir(d) if f.endswith('.cu'))
    flags = [f if not f.startswith('-I') else '-I' + os.path.abspath('include') for f in b.FLAGS]
    cmd = [b.NVCC] + b.ARCH + flags + list(extra) + srcs + ['-o', '_scratch/libgcb200_%s.so' % name]
    r = subprocess.run(cmd, capture_output=True, text=True)
    print(name, r.returncode, r.stderr[-500:] if r.returncode else '')
    shutil.rmtree('_scratch/src_' + name, ignore_errors=True)
