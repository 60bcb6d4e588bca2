import sys; sys.path.insert(0, '.')
import tools.slice_bench as sb
print(sb.run(50000, 128, 16, 1, 0, 0, reps=2))
