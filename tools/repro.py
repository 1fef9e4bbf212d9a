import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import test_gpu_kernels as T
case = sys.argv[1] if len(sys.argv) > 1 else "s1"
if case == "s1":
    print("worst", T._stage1_case(128, 8, 2, [150, 64, 97, 200, 33]))
elif case == "s1small":
    print("worst", T._stage1_case(128, 8, 2, [30]))
elif case == "s1two":
    print("worst", T._stage1_case(128, 8, 2, [64, 64]))
