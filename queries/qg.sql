SELECT l_partkey, SUM(l_extendedprice * (1 - l_discount)) AS revenue, SUM(l_quantity) AS sum_qty, COUNT(*) AS count_order
FROM lineitem WHERE l_shipdate >= DATE '1995-01-01' GROUP BY l_partkey
