import json, sys, time
sys.path.insert(0, "/root/repo")
from paper_2209_04579_b200 import tqp
ctx = tqp.default_context()
tables = {n: tqp.Table.generate(n, 10, 7, ctx=ctx) for n in sys.argv[1].split(",")}
plan = json.loads(open("/root/repo/paper_2209_04579_b200/plans/q1.opplan.json").read())
ex = tqp.Executor(plan, fuse=False, ctx=ctx)
for i in range(4):
    t = time.perf_counter(); ex.execute(tables); ctx.sync(); print("exec", (time.perf_counter()-t)*1e3)
for i in range(2):
    t = time.perf_counter(); ex.profile_execute(tables); ctx.sync(); print("prof", (time.perf_counter()-t)*1e3)
for i in range(2):
    t = time.perf_counter(); ex.execute(tables); ctx.sync(); print("exec", (time.perf_counter()-t)*1e3)
